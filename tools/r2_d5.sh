# GSE-8 slab kernel: quarter ranges exchanged by st.async + mbarrier instead of a cluster barrier
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "gse or GSE or blob or edge or quant" 2>&1 | tail -3
for r in 1 2 3; do echo "$(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"; done
