# attend: softmax warps between the decoder groups (SOFT_POS = groups below them): scheduler priority
set -x
HARAG_LIB=build/variants/wd2/libharag.so timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
for r in 1 2; do for v in default sp1 sp2 sp3 sp4; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
