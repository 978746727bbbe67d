# attend: unroll / prefetch distance combinations at 4 decoder groups
for r in 1 2 3; do for v in un4 un4pf2 un2 un4pf1; do
  export HARAG_LIB=build/variants/$v/libharag.so
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
