# pageable leg: copy-thread count sweep, interleaved (the leg varied 0.63-0.86 run to run on one box)
for r in 1 2; do for t in 9 6 12; do
  HARAG_COPY_THREADS=$t timeout 600 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); l=d['legs']['c2_tiered_pageable']; print('threads $t', l['value'], l['link']['achieved_GBps'], l['link']['frac'])"
done; done
