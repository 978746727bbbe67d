set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/pytest_attn.txt 2>&1; tail -3 gpurun_out/pytest_attn.txt
for v in default sleep0 sleep32 sleep160; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  for i in 1 2; do echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"; done
done > gpurun_out/attend_variants.txt 2>&1; cat gpurun_out/attend_variants.txt
unset HARAG_LIB
HARAG_LIB=build/variants/trace/libharag.so timeout 300 python tools/prof_attend.py 1 > gpurun_out/trace_b1.txt 2>&1
python tools/trace_attend.py gpurun_out/trace_b1.txt > gpurun_out/trace_b1_summary.txt 2>&1; cat gpurun_out/trace_b1_summary.txt
timeout 900 python bench.py --legs c2_tiered_pageable --no-e2e --no-cpu-baseline --no-per-scheme --steps 10 > gpurun_out/pageable.json 2> gpurun_out/pageable.err
python tools/show_bench.py gpurun_out/pageable.json 2>&1 | tail -4
