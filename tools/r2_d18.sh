# 4 decoder groups by default: attention parity, timing, sanitizers (attend and the host pool change ride along)
set -x
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for r in 1 2; do timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1; done
bash tools/sanitize.sh > gpurun_out/sanitize_run.log 2>&1; cat gpurun_out/sanitize/*.summary.txt
