# INT4 scale by Markstein (div15) + frcp_rn: exhaustive check, GPU suite, per-item timing
set -x
timeout 300 ./tests/csrc/markstein_check | tail -12
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for r in 1 2 3; do for s in INT4 INT8; do echo "$s $(timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done; done
