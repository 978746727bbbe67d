# attend S_FIRST ordering (PV_j queued after S_{j+2}): watchdog tests, parity, timing vs off, trace
set -x
HARAG_LIB=build/variants/wd/libharag.so timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in default sf0; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
unset HARAG_LIB
bash tools/r2_d30.sh; cat gpurun_out/d30_summary.txt
