set -x
mkdir -p gpurun_out
BB_REPS=3 timeout 900 ./tools/bounce_bench 1200 > gpurun_out/bounce_sweep.txt 2>&1
HARAG_LIB=build/variants/trace/libharag.so timeout 300 python tools/prof_attend.py 1 > gpurun_out/trace_b1.txt 2>&1
python tools/trace_attend.py gpurun_out/trace_b1.txt > gpurun_out/trace_b1_summary.txt 2>&1; cat gpurun_out/trace_b1_summary.txt
