set -x
for r in 1 2; do for v in default gseq2t128 gseq2t256 gseq1t256 gseq1t512; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done; done
for v in gseq2t256 gseq1t512; do HARAG_LIB=build/variants/$v/libharag.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "blobs or edge" 2>&1 | tail -1; done
