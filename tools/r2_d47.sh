# copy-window gaps without epochs (pinned leg)
HARAG_TIMELINE=gpurun_out/d47_pinned.txt timeout 900 python bench.py --legs c2_tiered_pinned --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme --epoch-every 0 > /dev/null 2>&1
grep h2d gpurun_out/d47_pinned.txt | head -12
