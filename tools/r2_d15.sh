# pageable leg with dynamically claimed 256 KiB bounce chunks: 4 runs
for r in 1 2 3 4; do
  timeout 600 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); l=d['legs']['c2_tiered_pageable']; print('dyn', l['value'], l['link']['achieved_GBps'], l['link']['frac'])"
done
