HARAG_HOST_PROF=1 timeout 900 python bench.py --legs c2_tiered_pinned --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>&1 >/dev/null | grep "host prof"
