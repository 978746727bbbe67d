# closing bench line after the staging-slot cap change
mkdir -p gpurun_out/fin5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin5/smoke.txt 2>&1; tail -1 gpurun_out/fin5/smoke.txt
timeout 1500 python bench.py > gpurun_out/fin5/bench_default.json 2> gpurun_out/fin5/bench_default.err; tail -c 200 gpurun_out/fin5/bench_default.json
