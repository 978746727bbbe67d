# attend decoder-group shape: 3 x 4 (default), 4 x 4, 2 x 8
for r in 1 2; do for v in default dg4 dg2w8; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
