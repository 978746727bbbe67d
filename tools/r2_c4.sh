# host bounce pipeline micro-benchmark, host topology, attend per-tile trace
set -x
mkdir -p gpurun_out
(nproc; lscpu | head -30; numactl -H 2>/dev/null | head; nvidia-smi topo -m 2>/dev/null | head; free -g) > gpurun_out/host.txt 2>&1
timeout 600 ./tools/bounce_bench 400 > gpurun_out/bounce_bench.txt 2>&1; cat gpurun_out/bounce_bench.txt
HARAG_LIB=build/variants/trace/libharag.so timeout 300 python tools/prof_attend.py 1 > gpurun_out/trace_b1.txt 2>&1
python tools/trace_attend.py gpurun_out/trace_b1.txt > gpurun_out/trace_b1_summary.txt 2>&1; cat gpurun_out/trace_b1_summary.txt
