# quantize ring at 32K tiles: 8 / 12 consumer warps; 24K tiles x 4 stages
for r in 1 2; do for v in default w8 w12 s4t24; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  for s in INT4 INT8; do echo "$v $(timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done
done; done
