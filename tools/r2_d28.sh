# quantize ring shape for INT4 / INT8: 32K-element tiles x 3 stages, 8 / 12 consumer warps
for r in 1 2; do for v in default t32s3 w8 w12; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  for s in INT4 INT8; do echo "$v $(timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done
done; done
