set -x
mkdir -p gpurun_out
for v in default gse_imad default gse_imad; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done
unset HARAG_LIB
HARAG_LIB=build/variants/gse_imad/libharag.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "blobs or edge" 2>&1 | tail -2
for v in default dec4 default dec4; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done
