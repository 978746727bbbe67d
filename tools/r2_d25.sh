# pageable leg: THP-advised pageable backing (default) vs 4 KiB pages, interleaved
for r in 1 2 3; do for thp in 1 0; do
  HARAG_HOST_THP=$thp timeout 600 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); l=d['legs']['c2_tiered_pageable']; print('thp=$thp', l['value'], l['link']['frac'], l['build_seconds'])"
done; done
grep -i AnonHuge /proc/meminfo
