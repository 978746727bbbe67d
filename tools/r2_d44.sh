# staging slots capped at 128 (default) vs 64: tiered legs, and the timeline of the default
for r in 1 2; do for v in default s64; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  timeout 900 python bench.py --legs c2_tiered_pinned,c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for n in ('c2_tiered_pinned','c2_tiered_pageable'):
  l=d['legs'][n]; print('$v', n, l['value'], l['ms_per_step'], l['link']['frac'], l['overlapped_roofline']['frac'])"
done; done
unset HARAG_LIB
HARAG_TIMELINE=gpurun_out/d44_timeline.txt timeout 900 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme > /dev/null 2>&1
grep h2d gpurun_out/d44_timeline.txt | head -12
