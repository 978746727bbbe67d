# A/B: round-1 tree vs HEAD on the headline (same box, alternating), MMA micro-benchmark, attend tests + ncu capture
set -x
mkdir -p gpurun_out
./tools/ubench/mma_lat > gpurun_out/mma_lat.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/pytest_attn.txt 2>&1; tail -3 gpurun_out/pytest_attn.txt
for i in 1 2; do
  (cd build/r1tree && timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-tiered --no-per-scheme > ../../gpurun_out/ab_r1_$i.json 2>../../gpurun_out/ab_r1_$i.err)
  timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --legs none --no-per-scheme > gpurun_out/ab_head_$i.json 2>/dev/null
done
timeout 600 python bench.py --attend > gpurun_out/attend.json 2> gpurun_out/attend.err; tail -c 1500 gpurun_out/attend.json
timeout 900 python bench.py --legs c2_ttft --no-e2e --no-cpu-baseline --no-per-scheme --steps 10 > gpurun_out/ttft.json 2> gpurun_out/ttft.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/r2_attend_b8 python tools/prof_attend.py 8 > gpurun_out/r2_attend_b8.log 2>&1
ls -la gpurun_out
