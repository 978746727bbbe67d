set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/pytest_c15.txt 2>&1; tail -3 gpurun_out/pytest_c15.txt
for i in 1 2 3; do timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1; done
timeout 900 python bench.py --legs c2_ttft --no-e2e --no-cpu-baseline --no-per-scheme --steps 10 > gpurun_out/ttft.json 2> gpurun_out/ttft.err; tail -c 1500 gpurun_out/ttft.json
