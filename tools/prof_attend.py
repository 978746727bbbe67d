"""Drive hr_attend for profiling: python tools/prof_attend.py [n_req] (C2 shape, paper ladder, 40 docs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_20878_b200 as hr  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
K_OVERRIDE = int(os.environ.get("HARAG_PROF_K", "10"))
L, H, T, D, k, n_docs, g, n_q = 32, 8, 512, 128, K_OVERRIDE, 40, 4, 32
h = hr.policy_count(synth.gen_requests(n_docs, 160, k, 1.1, seed=7), n_docs).astype(np.uint64)
ladder, taus = ("INT8", "FP8E4M3", "FP8E5M2", "GSE8"), (0.1, 0.1, 0.1)
total = sum(hr.item_bytes(int(s), L=L, H=H, D=D, T=T) for s in hr.policy_assign(h, ladder, taus))
st = hr.Store(L=L, H=H, D=D, T=T, ladder=ladder, taus=taus, hbm_budget=total + (1 << 20), keep_backing=False)
st.build(n_docs, h, lambda d, kp, vp, s: (synth.gen_item_device(kp, L, H, T, D, d, 0, stream=s),
                                          synth.gen_item_device(vp, L, H, T, D, d, 1, stream=s)))
reqs = synth.gen_requests(n_docs, B, k, 1.1, seed=3).astype(np.uint32)
q = torch.from_numpy(synth.gen_query(B, L, H * g, n_q, D).view(np.int16)).cuda()
o = torch.empty_like(q)
for _ in range(3):
    st.attend(reqs, q, o, n_q, g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    st.attend(reqs, q, o, n_q, g)
e1.record()
e1.synchronize()
print(f"attend: {e0.elapsed_time(e1) / 5:.3f} ms per batch of {B}")
