set -x
mkdir -p gpurun_out
for r in 1 2; do for v in default gseq8 gseq2; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done; done
HARAG_LIB=build/variants/gseq8/libharag.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "blobs or edge" 2>&1 | tail -2
