# INT4 correction-free common case: exhaustive/sampled check, GPU parity, timing
set -x
timeout 600 ./tests/csrc/markstein_check | tail -8
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2 3; do echo "$(timeout 120 python tools/prof_quant.py INT4 64 2>&1 | tail -1)"; done
