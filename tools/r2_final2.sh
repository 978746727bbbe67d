# Round-2 closing validation + profiling pass on one B200 (summaries copied to profiles/round2/)
set -x
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin/pytest_gpu.txt 2>&1; tail -3 gpurun_out/fin/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.txt 2>&1; tail -2 gpurun_out/fin/smoke.txt
timeout 1500 python bench.py > gpurun_out/fin/bench_default.json 2> gpurun_out/fin/bench_default.err; tail -c 300 gpurun_out/fin/bench_default.json
timeout 600 python bench.py --attend > gpurun_out/fin/attend.json 2> gpurun_out/fin/attend.err; tail -c 300 gpurun_out/fin/attend.json
timeout 900 python bench.py --ablation > gpurun_out/fin/ablation.json 2> gpurun_out/fin/ablation.err; tail -c 300 gpurun_out/fin/ablation.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err; tail -c 300 gpurun_out/fin/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/fin/launches.csv \
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --legs none --no-per-scheme > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:assemble_kv -s 3 -c 2 --csv --log-file gpurun_out/fin/traffic.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --legs none --no-per-scheme > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assemble_kv -s 3 -c 1 -o gpurun_out/fin/assemble_c2 \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --legs none --no-per-scheme > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/fin/attend_b8 python tools/prof_attend.py 8 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gse_slab -s 1 -c 1 -o gpurun_out/fin/gse_slab python tools/prof_quant.py GSE8 16 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 1 -c 1 -o gpurun_out/fin/q_int4 python tools/prof_quant.py INT4 16 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 1 -c 1 -o gpurun_out/fin/q_int8 python tools/prof_quant.py INT8 16 > /dev/null 2>&1
ls -la gpurun_out/fin
