"""Per-buffer H2D bandwidth of freshly pinned host buffers (physical placement probe):
python tools/pin_probe.py [n_buffers] [MiB]"""
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 16
bufs = [torch.empty(mib << 20, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
for b in bufs:
    b.fill_(1)
dst = torch.empty(mib << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for i, b in enumerate(bufs):
    best = 1e9
    for _ in range(5):
        e0.record()
        dst.copy_(b, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res.append((mib << 20) / (best / 1e3) / 1e9)
print(" ".join(f"{g:.1f}" for g in res))
