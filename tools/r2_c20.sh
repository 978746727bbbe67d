set -x
mkdir -p gpurun_out
for r in 1 2; do for v in default main4 rare1 main4rare1; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done; done
unset HARAG_LIB
HARAG_SINGLE_DEVICE=1 HARAG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --legs none --no-per-scheme --no-e2e > gpurun_out/n2_gloo.json 2> gpurun_out/n2_gloo.err; tail -c 800 gpurun_out/n2_gloo.json; tail -5 gpurun_out/n2_gloo.err
