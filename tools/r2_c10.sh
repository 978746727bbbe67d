set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_attention.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/pytest_c10.txt 2>&1; tail -3 gpurun_out/pytest_c10.txt
for v in default softone default softone; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done > gpurun_out/attend_variants3.txt 2>&1
unset HARAG_LIB
for d in 0 25 10 50; do
  echo "dyn=$d $(HARAG_ASM_DYN=$d timeout 600 python tools/lat_probe.py 128 2>&1 | head -1)"
done > gpurun_out/lat_dyn.txt 2>&1
for d in 0 25; do
  HARAG_ASM_DYN=$d timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --legs none --no-per-scheme > gpurun_out/ab_dyn$d.json 2>/dev/null
done
cat gpurun_out/attend_variants3.txt gpurun_out/lat_dyn.txt
HARAG_LIB=build/variants/trace/libharag.so timeout 300 python tools/prof_attend.py 1 > gpurun_out/trace_b1.txt 2>&1
python tools/trace_attend.py gpurun_out/trace_b1.txt
