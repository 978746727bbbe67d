# final state of the round: GPU suite, smoke, default bench line, reference arm
set -x
mkdir -p gpurun_out/fin4
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin4/pytest_gpu.txt 2>&1; tail -2 gpurun_out/fin4/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4/smoke.txt 2>&1; tail -1 gpurun_out/fin4/smoke.txt
timeout 1500 python bench.py > gpurun_out/fin4/bench_default.json 2> gpurun_out/fin4/bench_default.err; tail -c 200 gpurun_out/fin4/bench_default.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin4/bench_ref.json 2> gpurun_out/fin4/bench_ref.err; tail -c 200 gpurun_out/fin4/bench_ref.json
