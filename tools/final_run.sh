set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 400 gpurun_out/bench_default.json
timeout 600 python bench.py --attend > gpurun_out/attend.json 2> gpurun_out/attend.err; cat gpurun_out/attend.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/att_final python tools/prof_attend.py 8 > /dev/null 2>&1
ls gpurun_out | tail -5
