"""Drive the quantize kernels for profiling: python tools/prof_quant.py SCHEME [n_docs]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_20878_b200 as hr  # noqa: E402
import synth  # noqa: E402

scheme = sys.argv[1]
n_docs = int(sys.argv[2]) if len(sys.argv) > 2 else 20
L, H, T, D = 32, 8, 512, 128
src = torch.empty(2, L * H * T * D, dtype=torch.int16, device="cuda")
synth.gen_item_device(src[0].data_ptr(), L, H, T, D, 0, 0)
synth.gen_item_device(src[1].data_ptr(), L, H, T, D, 0, 1)
item = hr.item_bytes(scheme, L=L, H=H, D=D, T=T)
st = hr.Store(L=L, H=H, D=D, T=T, ladder=(scheme,), taus=(), keep_backing=False,
              hbm_budget=2 * n_docs * item + (1 << 20))
st.build_begin(n_docs, np.zeros(2 * n_docs, np.uint64))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for d in range(n_docs):
    st.build_put(d, src[0], src[1])
e1.record()
st.build_end()
ms = e0.elapsed_time(e1)
print(f"{scheme}: {1e3 * ms / (2 * n_docs):.2f} us/item, "
      f"{2 * n_docs * (L * H * T * D * 2 + item) / (ms / 1e3) / 1e9:.0f} GB/s")
