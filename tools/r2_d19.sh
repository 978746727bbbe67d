# attend knobs at 4 decoder groups
for r in 1 2; do for v in default ga1 pf8 pf2 un4; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
