set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --legs c2_tiered_pageable --no-e2e --no-cpu-baseline --no-per-scheme --steps 20 > gpurun_out/pageable.json 2> gpurun_out/pageable.err
python tools/show_bench.py gpurun_out/pageable.json 2>&1 | tail -3
