set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_c11.txt 2>&1; tail -3 gpurun_out/pytest_c11.txt
for d in 0 25 0 25; do
  for s in INT8 INT4; do echo "qdyn=$d $(HARAG_Q_DYN=$d timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done
done > gpurun_out/q_dyn.txt 2>&1; cat gpurun_out/q_dyn.txt
