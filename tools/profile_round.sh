# Round profiling pass on one B200 (outputs under gpurun_out/; summaries are copied to profiles/ by hand)
set -x
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tiered --no-per-scheme > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 3 -c 1 -o gpurun_out/prof_quant_int8 python tools/prof_quant.py INT8 8 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 6 -c 2 -o gpurun_out/prof_quant_gse python tools/prof_quant.py GSE8 8 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 3 -c 1 -o gpurun_out/prof_quant_int4 python tools/prof_quant.py INT4 8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/prof_attend python tools/prof_attend.py 1 > /dev/null 2>&1
ls -la gpurun_out/
