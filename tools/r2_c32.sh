set -x
for i in 1 2; do
timeout 900 python bench.py --legs c2_tiered_pageable --no-e2e --no-cpu-baseline --no-per-scheme --steps 20 > gpurun_out/pageable_$i.json 2> gpurun_out/pageable.err
python tools/show_bench.py gpurun_out/pageable_$i.json 2>&1 | tail -1
done
