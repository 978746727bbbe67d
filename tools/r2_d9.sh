# attend: baseline timing (3 runs) and one ncu --set full capture with source for an opcode histogram
for r in 1 2 3; do timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/d9_attend python tools/prof_attend.py 8 > gpurun_out/d9_ncu.log 2>&1
