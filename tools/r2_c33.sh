set -x
for r in 1 2; do for v in default qtilegrp qw24 qs6; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  for s in INT8 INT4; do echo "$v $(timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done
done; done
