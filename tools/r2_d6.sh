# GSE-8 slab kernel cluster shape after the st.async exchange
for r in 1 2; do for v in default q4t256 q4t128 q2t128; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done; done
