# copy-window gaps vs hardware work queues: CUDA_DEVICE_MAX_CONNECTIONS=32 (default 8)
CUDA_DEVICE_MAX_CONNECTIONS=32 HARAG_TIMELINE=gpurun_out/d48_pinned.txt timeout 900 python bench.py --legs c2_tiered_pinned,c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for n in ('c2_tiered_pinned','c2_tiered_pageable'):
  l=d['legs'][n]; print('conn32', n, l['value'], l['ms_per_step'], l['link']['frac'], l['overlapped_roofline']['frac'])"
grep h2d gpurun_out/d48_pinned.txt | head -10
