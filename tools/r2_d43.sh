# tiered legs: cost of the epochs (re-rank, re-place, promotions) inside the timed steps
for ee in 8 0; do
  timeout 900 python bench.py --legs c2_tiered_pinned,c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme --epoch-every $ee 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for n in ('c2_tiered_pinned','c2_tiered_pageable'):
  l=d['legs'][n]; print('epoch_every=$ee', n, l['ms_per_step'], l['link']['frac'], l['overlapped_roofline']['frac'], l.get('migrations'))"
done
HARAG_TIMELINE=gpurun_out/d43_timeline.txt timeout 900 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme > /dev/null 2>&1
ls -la gpurun_out/d43_timeline.txt; head -c 3000 gpurun_out/d43_timeline.txt
