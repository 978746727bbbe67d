# ncu --set full with source: INT4 encode (ring kernel) and GSE-8 slab kernel after the INT4 change
ncu --set full --clock-control none --import-source on -k regex:quantize_batch -s 1 -c 1 -o gpurun_out/d2_int4 python tools/prof_quant.py INT4 16 > gpurun_out/d2_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gse_slab -s 1 -c 1 -o gpurun_out/d2_gse python tools/prof_quant.py GSE8 16 > gpurun_out/d2_ncu2.log 2>&1
ls -la gpurun_out
