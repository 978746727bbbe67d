# attend per-tile trace (CTA 0) at four decoder groups
HARAG_LIB=build/variants/trace/libharag.so timeout 300 python tools/prof_attend.py 8 > gpurun_out/d30_trace.txt 2>&1
python tools/trace_attend.py gpurun_out/d30_trace.txt 20 76 > gpurun_out/d30_summary.txt 2>&1
