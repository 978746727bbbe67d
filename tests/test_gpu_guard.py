"""GPU parity of the value-distribution guard (R29; SURVEY §8(f) item 4 extra) against
oracle/guard.py: the per-item statistics of hr_guard_stats (flush count exact, max |x| bit-exact), the
schemes a guard-enabled hr_build_store assigns, and the assembled KV of that store bit-exact against the
oracle store built with the oracle's guarded schemes."""
import numpy as np
import pytest

import synth
from oracle import guard, hotness, numerics
from oracle import store as ost

pytestmark = pytest.mark.gpu

NAMES = {"PASS16": ost.PASS16, "INT8": ost.INT8, "FP8E4M3": ost.FP8E4M3, "FP8E5M2": ost.FP8E5M2,
         "GSE8": ost.GSE8, "INT4": ost.INT4}
PAPER = ("INT8", "FP8E4M3", "FP8E5M2", "GSE8")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def bits_of(v: float, dtype: str) -> int:
    x = np.array([v], dtype=np.float32)
    return int(numerics.f32_to_bf16(x)[0]) if dtype == "bf16" else int(x.astype(np.float16).view(np.uint16)[0])


def make_items(n_docs, L, H, T, D, dtype, seed):
    """Synthetic items (all heads) with injected hazards: tiny values (GSE-8 flush), magnitudes past the
    FP8 E4M3 / E5M2 ranges, 16-bit subnormals."""
    rng = np.random.default_rng(seed)
    items = {}
    for doc in range(n_docs):
        for kind in range(2):
            it = synth.gen_item(L, H, T, D, doc, kind, dtype=dtype).copy()
            r = rng.random()
            l, h = int(rng.integers(L)), int(rng.integers(H))
            pos = rng.integers(0, T * D, size=3)
            flat = it[l, h].reshape(-1)
            if r < 0.3:
                flat[pos] = bits_of(2.0 ** -30 if dtype == "bf16" else 2.0 ** -24, dtype)
            elif r < 0.45:
                flat[pos[0]] = bits_of(1000.0, dtype)
            elif r < 0.55 and dtype == "bf16":
                flat[pos[0]] = bits_of(60000.0 * 2, dtype)
            elif r < 0.65:
                flat[pos] = 0x0001  # smallest positive subnormal
            items[(doc, kind)] = it
    return items


@pytest.mark.parametrize("dtype,gse", [("bf16", (4, 3)), ("bf16", (2, 5)), ("fp16", (4, 3)), ("fp16", (3, 4))])
def test_guard_stats_match_oracle(torch_cuda, dtype, gse):
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D = 2, 4, 64, 64
    items = make_items(6, L, H, T, D, dtype, seed=3)
    stats = torch.zeros((len(items), 2), dtype=torch.int64, device="cuda")
    srcs = []
    for i, it in enumerate(items.values()):
        src = torch.from_numpy(it.view(np.int16)).cuda()
        srcs.append(src)
        hr.guard_stats(src, stats[i], L=L, H=H, D=D, T=T, dtype=dtype, gse=gse)
    got = stats.cpu().numpy().view(np.uint64)
    for i, it in enumerate(items.values()):
        fl, am = guard.guard_stats(it, dtype, *gse)
        assert int(got[i, 0]) == fl, (i, int(got[i, 0]), fl)
        assert int(got[i, 1]) == int(np.array([am], np.float32).view(np.uint32)[0]), (i, hex(int(got[i, 1])), am)


@pytest.mark.parametrize("gse", [(4, 3), (2, 5)])
def test_store_with_guard_matches_oracle(torch_cuda, gse):
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D, n_docs, k, dtype = 2, 2, 64, 64, 16, 4, "bf16"
    taus = (0.2, 0.2, 0.2)
    items = make_items(n_docs, L, H, T, D, dtype, seed=11)
    dev = {key: torch.from_numpy(v.view(np.int16)).cuda() for key, v in items.items()}
    prof = synth.gen_requests(n_docs, 64, k, 1.1, seed=7)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype=dtype, gse_e=gse[0], gse_m=gse[1])
    ladder_ids = [NAMES[s] for s in PAPER]
    a1 = hotness.assign_schemes(h.tolist(), ladder_ids, taus)
    stats = [guard.guard_stats(items[(i // 2, i % 2)], dtype, *gse) for i in range(2 * n_docs)]
    want = guard.guard_schemes(a1, stats, ladder_ids)
    assert want != a1  # the injected hazards move some items

    sizes = [lay.item_bytes(s) for s in want]
    st = hr.Store(L=L, H=H, D=D, T=T, dtype=dtype, gse=gse, ladder=PAPER, taus=taus, hbm_budget=sum(sizes) + 4096,
                  guard=True)

    def src(doc, kp, vp, stream):
        # the library's buffers as torch tensors (zero-copy, __cuda_array_interface__); the copies run on
        # torch's current stream = the legacy default stream the build uses (stream None)
        n = L * H * T * D
        for p, key in ((kp, (doc, 0)), (vp, (doc, 1))):
            torch.as_tensor(hr._DevArray(p, n, "<i2"), device="cuda").copy_(dev[key].view(-1))

    st.build(n_docs, h, src)
    got = [st.item_info(i)[0] for i in range(2 * n_docs)]
    assert got == want
    ora = ost.OracleStore(lay, ladder_ids, taus)
    ora.build(n_docs, h, lambda d, kind: items[(d, kind)], schemes=want)
    reqs = synth.gen_requests(n_docs, 6, k, 1.1, seed=2)
    nb = st.kv_bytes(k)
    ko = [torch.empty(nb // 2, dtype=torch.int16, device="cuda") for _ in reqs]
    vo = [torch.empty(nb // 2, dtype=torch.int16, device="cuda") for _ in reqs]
    st.assemble(reqs, ko, vo)
    torch.cuda.synchronize()
    for r, req in enumerate(reqs):
        K, V = ora.assemble(list(req))
        assert np.array_equal(ko[r].cpu().numpy().view(np.uint16).reshape(K.shape), K), r
        assert np.array_equal(vo[r].cpu().numpy().view(np.uint16).reshape(V.shape), V), r
    st.close()
