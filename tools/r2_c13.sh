set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_guard.py tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/pytest_c13.txt 2>&1; tail -30 gpurun_out/pytest_c13.txt
for i in 1 2; do timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1; done
