# placement-probed bounce buffers: GPU suite, pageable leg x4, bounce probe stats
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2 3 4; do
  timeout 600 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); l=d['legs']['c2_tiered_pageable']; print('probed', l['value'], l['link']['frac'], l['build_seconds'])"
done
