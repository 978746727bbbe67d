ncu --metrics gpu__time_duration.sum --clock-control none -c 60 python tools/prof_quant.py INT4 16 > gpurun_out/d3_list.log 2>&1
env | grep -i -E "harag|cuda|ncu" > gpurun_out/d3_env.log
ldd paper_2510_20878_b200/libharag.so >> gpurun_out/d3_env.log
