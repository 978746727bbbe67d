# attend: P rounded half-up by an FMA-pipe IMAD + PRMT (default) / VIADD + PRMT / F2FP
set -x
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in default viadd pf0; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
