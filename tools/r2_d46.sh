# copy-window gaps: pinned leg timeline and host-side phase profile of the pageable leg
HARAG_TIMELINE=gpurun_out/d46_pinned.txt timeout 900 python bench.py --legs c2_tiered_pinned --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme > /dev/null 2>&1
grep h2d gpurun_out/d46_pinned.txt | head -12
HARAG_HOST_PROF=1 timeout 900 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>&1 >/dev/null | grep "host prof"
