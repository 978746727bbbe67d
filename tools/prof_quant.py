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
NS = 16  # distinct source docs (16 x 67 MB >> 126 MB L2), cycled
src = torch.empty(NS, 2, L * H * T * D, dtype=torch.int16, device="cuda")
for i in range(NS):
    synth.gen_item_device(src[i, 0].data_ptr(), L, H, T, D, i, 0)
    synth.gen_item_device(src[i, 1].data_ptr(), L, H, T, D, i, 1)
item = hr.item_bytes(scheme, L=L, H=H, D=D, T=T)
st = hr.Store(L=L, H=H, D=D, T=T, ladder=(scheme,), taus=(), keep_backing=False,
              hbm_budget=2 * n_docs * item + (1 << 20))
st.build_begin(n_docs, np.zeros(2 * n_docs, np.uint64))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
QB = int(os.environ.get("HARAG_PUT_BATCH", "16"))  # docs per hr_build_put_batch (one launch)
st.build_put_batch(range(min(QB, n_docs)), [src[i % NS, 0] for i in range(min(QB, n_docs))],
                   [src[i % NS, 1] for i in range(min(QB, n_docs))])  # warm-up (module load, first touch)
torch.cuda.synchronize()
e0.record()
for d in range(0, n_docs, QB):
    nd = min(QB, n_docs - d)
    st.build_put_batch(range(d, d + nd), [src[(d + i) % NS, 0] for i in range(nd)],
                       [src[(d + i) % NS, 1] for i in range(nd)])
e1.record()
st.build_end()
ms = e0.elapsed_time(e1)
print(f"{scheme}: {1e3 * ms / (2 * n_docs):.2f} us/item, "
      f"{2 * n_docs * (L * H * T * D * 2 + item) / (ms / 1e3) / 1e9:.0f} GB/s")
