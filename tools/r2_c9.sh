set -x
mkdir -p gpurun_out
timeout 600 python tools/lat_probe.py 256 > gpurun_out/lat_probe.txt 2>&1; head -3 gpurun_out/lat_probe.txt
