set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "blobs or edge or ties or nan" > gpurun_out/pytest_q.txt 2>&1; tail -3 gpurun_out/pytest_q.txt
for v in default gse_alu default gse_alu; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_quant.py GSE8 64 2>&1 | tail -1)"
done > gpurun_out/q_variants.txt 2>&1; cat gpurun_out/q_variants.txt
unset HARAG_LIB
for s in INT4 INT8; do echo "$(timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done >> gpurun_out/q_variants.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gse_slab -s 40 -c 1 -o gpurun_out/r2_gse_slab python tools/prof_quant.py GSE8 16 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 3 -c 1 -o gpurun_out/r2_q_int4 python tools/prof_quant.py INT4 16 > /dev/null 2>&1
cat gpurun_out/q_variants.txt
