# attend decoder groups: 4 x 4 vs 5 x 4 vs 4 x 4 with 3 S buffers
for r in 1 2; do for v in dg4 dg5 dg4sb3; do
  export HARAG_LIB=build/variants/$v/libharag.so
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
