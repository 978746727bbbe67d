set -x
HARAG_HOST_PROF=1 timeout 600 python tools/lat_probe.py 128 2>&1 | grep -E "calls|host prof"
for c in 4 16 32; do echo "chunks=$c $(HARAG_ASM_CHUNKS=$c timeout 600 python tools/lat_probe.py 128 2>&1 | head -1)"; done
for d in 35 15; do echo "dyn=$d $(HARAG_ASM_DYN=$d timeout 600 python tools/lat_probe.py 128 2>&1 | head -1)"; done
