set -x
for r in 1 2; do for v in default inl24 inl0; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 600 python tools/lat_probe.py 128 2>&1 | head -1)"
done; done
