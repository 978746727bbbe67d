# attend: P buffers decoupled from S buffers (kPB = 3): watchdog build first (a deadlock traps instead of hanging),
# then the default build's parity tests and timing vs kPB = 2 / 4
set -x
HARAG_LIB=build/variants/wd/libharag.so timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in default pb2 pb4; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
