# GSE-8 slab kernel: part source in TMA pieces with a barrier each (range pass overlaps the load)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "gse or GSE or blob or edge or quant or guard" 2>&1 | tail -2
for r in 1 2 3; do for v in default c1 c2 c8; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done; done
