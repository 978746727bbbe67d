# quantize ring with 32K-element tiles x 3 stages: full GPU suite and per-scheme timing
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for s in INT4 INT8 GSE8 PASS16 FP8E4M3; do echo "$s $(timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done; done
