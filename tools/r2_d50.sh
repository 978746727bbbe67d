# pinned-source copies enqueued ahead of launch A (default) vs after (HARAG_EARLY_COPIES=0)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for e in 1 0; do
  HARAG_EARLY_COPIES=$e HARAG_TIMELINE=gpurun_out/d50_e$e.txt timeout 900 python bench.py --legs c2_tiered_pinned,c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for n in ('c2_tiered_pinned','c2_tiered_pageable'):
  l=d['legs'][n]; print('early=$e', n, l['value'], l['ms_per_step'], l['link']['frac'], l['overlapped_roofline']['frac'])"
  grep h2d gpurun_out/d50_e$e.txt | head -8
done
