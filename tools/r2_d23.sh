# attend at four decoder groups: softmax warps on the highest ids; three operand buffers
for r in 1 2; do for v in default softlast ob3; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
