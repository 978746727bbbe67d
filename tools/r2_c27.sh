set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tail_balanced" 2>&1 | tail -2
HARAG_LIB=build/variants/trace/libharag.so timeout 300 python tools/prof_attend.py 1 > gpurun_out/trace_b1.txt 2>&1
python tools/trace_attend.py gpurun_out/trace_b1.txt
