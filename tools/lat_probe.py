"""Single-request assemble latency, per call: python tools/lat_probe.py [n_calls]
C2 HBM-resident store (as bench.py); per call the library's entry->done time (hr_last_call_ms) and the
kernel-only time (library events around the launch), with the request's scheme mix, so the p50 / p99
spread can be attributed (request content vs launch / host jitter)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_20878_b200 as hr  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
args = argparse.Namespace(gpus=1)
ctx = bench.Ctx(args)
torch = ctx.torch
wl = dict(bench.WORKLOADS["c2"])
st, h, schemes, _, _ = bench.build_store(ctx, wl)
reqs = synth.gen_requests(wl["n_docs"], wl["batch"], wl["k"], wl["s"], seed=1)
kvb = st.kv_bytes(wl["k"])
ko = [torch.empty(kvb // 2, dtype=torch.int16, device="cuda")]
vo = [torch.empty(kvb // 2, dtype=torch.int16, device="cuda")]
rows = []
for i in range(n + 8):
    req = reqs[i % len(reqs):i % len(reqs) + 1]
    st.reset_stats()
    st.set_timing(True, calls=True)
    st.assemble(req, ko, vo, stream=ctx.stream)
    call = st.last_call_ms() * 1e3
    s = st.stats()
    kern = s["kernel_ms"] * 1e3
    if i >= 8:
        sch = [int(schemes[2 * d + kd]) for d in req[0] for kd in (0, 1)]
        rows.append((i % len(reqs), call, kern, sum(1 for x in sch if x == hr.GSE8)))
st.set_timing(False, calls=False)
a = np.array(rows)
print(f"calls {len(a)}: call p50 {np.percentile(a[:, 1], 50):.1f} p99 {np.percentile(a[:, 1], 99):.1f} max {a[:, 1].max():.1f} us; "
      f"kernel p50 {np.percentile(a[:, 2], 50):.1f} p99 {np.percentile(a[:, 2], 99):.1f} us; "
      f"call - kernel p50 {np.percentile(a[:, 1] - a[:, 2], 50):.1f} p99 {np.percentile(a[:, 1] - a[:, 2], 99):.1f}")
for r in range(len(reqs)):
    m = a[a[:, 0] == r]
    print(f"req {r:2d} gse_items {int(m[0, 3]):2d}: call {m[:, 1].mean():6.1f} (min {m[:, 1].min():6.1f} max {m[:, 1].max():6.1f}) "
          f"kernel {m[:, 2].mean():6.1f}")
st.close()  # prints the HARAG_HOST_PROF breakdown when set
