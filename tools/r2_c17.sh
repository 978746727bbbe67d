set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/pytest_c17.txt 2>&1; tail -40 gpurun_out/pytest_c17.txt
for s in MXFP8 FP8E4M3; do timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1; done
