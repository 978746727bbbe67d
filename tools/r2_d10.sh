# attend: linear decoder chunk addressing + 3-op FP8 pair decode; parity (attention tests) and timing
set -x
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3
for r in 1 2 3 4; do timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1; done
