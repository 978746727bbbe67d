# quantize kernels on one B200: per-item throughput (host-launched build_put loop) and ncu launch list
for s in PASS16 INT8 FP8E4M3 GSE8 INT4; do
  python tools/prof_quant.py $s 100 > gpurun_out/q_$s.txt 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/qncu_$s.csv python tools/prof_quant.py $s 10 > /dev/null 2>&1
done
