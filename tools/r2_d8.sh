# GSE-8 A/B, 5 runs each, interleaved
for r in 1 2 3 4 5; do for v in default imad imad2; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done; done
