# one ncu --set full capture per quantize variant (INT8, INT4, GSE-8 encode, GSE-8 range)
ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 3 -c 1 -o gpurun_out/qfull_int8 python tools/prof_quant.py INT8 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 3 -c 1 -o gpurun_out/qfull_int4 python tools/prof_quant.py INT4 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 6 -c 2 -o gpurun_out/qfull_gse python tools/prof_quant.py GSE8 6 > /dev/null 2>&1
