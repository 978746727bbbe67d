# attend changes (split, DUMP template, cursors): tests + timing; assemble inline-descriptor A/B; TTFT; sanitizers
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/pytest_attn.txt 2>&1; tail -3 gpurun_out/pytest_attn.txt
for i in 1 2 3; do python tools/prof_attend.py 8; done > gpurun_out/prof_attend.txt 2>&1; cat gpurun_out/prof_attend.txt
for i in 1 2; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --legs none --no-per-scheme > gpurun_out/ab_head_$i.json 2>/dev/null
  HARAG_LIB=build/variants/noinline/libharag.so timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --legs none --no-per-scheme > gpurun_out/ab_noinl_$i.json 2>/dev/null
done
timeout 900 python bench.py --legs c2_ttft --no-e2e --no-cpu-baseline --no-per-scheme --steps 10 > gpurun_out/ttft.json 2> gpurun_out/ttft.err
timeout 2400 bash tools/sanitize.sh > gpurun_out/sanitize_run.txt 2>&1
ls -la gpurun_out gpurun_out/sanitize
