# quantize throughput per scheme for each tuning variant under build/variants/
for v in build/variants/*/; do
  n=$(basename $v)
  for s in PASS16 INT8 FP8E4M3 GSE8 INT4; do
    echo "$n $(HARAG_LIB=$v/libharag.so python tools/prof_quant.py $s 48 2>&1 | tail -1)"
  done
done
