# attend with kPB = 3 (S_FIRST removed): full GPU suite, timing
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2 3; do timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1; done
