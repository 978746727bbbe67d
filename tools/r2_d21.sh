# attend census at 4 decoder groups, unroll 4, prefetch 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/d21_attend python tools/prof_attend.py 8 > gpurun_out/d21_ncu.log 2>&1
