# pageable leg variance (3 runs) + INT4 tree statistics timing
nproc; cat /proc/cpuinfo | grep "model name" | head -1; free -g | head -2
for r in 1 2 3; do timeout 600 python bench.py --legs c2_tiered_pageable --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-per-scheme 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); l=d['legs']['c2_tiered_pageable']; print('pageable', l['value'], l['link'])"; done
for r in 1 2 3; do echo "$(timeout 120 python tools/prof_quant.py INT4 64 2>&1 | tail -1)"; done
