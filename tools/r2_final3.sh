# closing bench line after the bounce probe / THP / ring-tile changes, and the INT4 ncu refresh
set -x
mkdir -p gpurun_out/fin3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3/smoke.txt 2>&1; tail -1 gpurun_out/fin3/smoke.txt
timeout 1500 python bench.py > gpurun_out/fin3/bench_default.json 2> gpurun_out/fin3/bench_default.err; tail -c 300 gpurun_out/fin3/bench_default.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 1 -c 1 -o gpurun_out/fin3/q_int4 python tools/prof_quant.py INT4 16 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 1 -c 1 -o gpurun_out/fin3/q_int8 python tools/prof_quant.py INT8 16 > /dev/null 2>&1
