# pageable leg: alone vs after the pinned leg in the same process (the default bench line runs them in sequence)
for r in 1 2; do
  timeout 900 python bench.py --legs c2_tiered_pinned,c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); l=d['legs']['c2_tiered_pageable']; print('after-pinned', l['value'], l['link']['frac'])"
  timeout 600 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); l=d['legs']['c2_tiered_pageable']; print('alone', l['value'], l['link']['frac'])"
done
free -g | head -2; cat /sys/kernel/mm/transparent_hugepage/enabled; grep -i huge /proc/meminfo
