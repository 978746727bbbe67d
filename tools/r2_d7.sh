# GSE-8: signed-min range pass (default) and FMA-pipe table addressing (imad = old range pass, imad2 = new)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "gse or GSE or blob or edge or quant or guard" 2>&1 | tail -3
for r in 1 2; do for v in default imad imad2; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done; done
