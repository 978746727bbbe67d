"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, on the
same seeded inputs.  Packed blobs, placement and assembled KV are compared bit
for bit (R3: both sides take every decision in fp32 RNE)."""
import numpy as np
import pytest

import synth
from oracle import hotness, placement
from oracle import store as ost

pytestmark = pytest.mark.gpu

NAMES = {"PASS16": ost.PASS16, "INT8": ost.INT8, "FP8E4M3": ost.FP8E4M3, "FP8E5M2": ost.FP8E5M2,
         "GSE8": ost.GSE8, "INT4": ost.INT4, "MXFP8": ost.MXFP8}
PAPER = ("INT8", "FP8E4M3", "FP8E5M2", "GSE8")
NORTH = ("PASS16", "INT8", "INT4")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def gpu_source(L, H, T, D, dtype, seed=synth.CORPUS_SEED):
    def src(doc, kp, vp, stream):
        synth.gen_item_device(kp, L, H, T, D, doc, 0, dtype=dtype, seed=seed, stream=stream)
        synth.gen_item_device(vp, L, H, T, D, doc, 1, dtype=dtype, seed=seed, stream=stream)
    return src


def make_pair(torch, *, L, H, T, D, n_docs, ladder, taus, dtype="bf16", group=0, gse=(4, 3),
              hbm_items=None, pin_items=0, rank=0, world=1, hot_seed=7, backing_pinned=False,
              keep_backing=True, decay_shift=1):
    """Build the GPU store and the oracle store on the same inputs."""
    import paper_2510_20878_b200 as hr
    prof = synth.gen_requests(n_docs, 4 * n_docs, min(4, n_docs), 1.1, seed=hot_seed)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype=dtype, group=group, gse_e=gse[0], gse_m=gse[1],
                     rank=rank, world=world)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in ladder], taus)
    sizes = [lay.item_bytes(s) for s in schemes]
    order = hotness.rank_items(h)
    if hbm_items is None:
        hbm_budget = sum(sizes) + 4096
    else:
        hbm_budget = sum(sizes[i] for i in order[:hbm_items])
    pin_budget = sum(sizes[i] for i in order[len(order) if hbm_items is None else hbm_items:][:pin_items])
    st = hr.Store(L=L, H=H, D=D, T=T, dtype=dtype, group=group, gse=gse, ladder=ladder, taus=taus,
                  hbm_budget=hbm_budget, pin_budget=pin_budget, rank=rank, world=world,
                  backing_pinned=backing_pinned, keep_backing=keep_backing, decay_shift=decay_shift)
    st.build(n_docs, h, gpu_source(L, H, T, D, dtype))
    ora = ost.OracleStore(lay, [NAMES[s] for s in ladder], taus)
    ora.build(n_docs, h, lambda d, k: synth.gen_item(L, H, T, D, d, k, heads=lay.heads, dtype=dtype))
    return st, ora, lay, h, sizes


def alloc_out(torch, st, n_req, k):
    nb = st.kv_bytes(k)
    ko = [torch.full((nb // 2,), 0x7FFF, dtype=torch.int16, device="cuda") for _ in range(n_req)]
    vo = [torch.full((nb // 2,), 0x7FFF, dtype=torch.int16, device="cuda") for _ in range(n_req)]
    return ko, vo


def check_requests(torch, st, ora, lay, reqs):
    k = reqs.shape[1]
    ko, vo = alloc_out(torch, st, len(reqs), k)
    st.assemble(reqs, ko, vo)
    torch.cuda.synchronize()
    for r, req in enumerate(reqs):
        K, V = ora.assemble(list(req))
        gk = ko[r].cpu().numpy().view(np.uint16).reshape(K.shape)
        gv = vo[r].cpu().numpy().view(np.uint16).reshape(V.shape)
        assert np.array_equal(gk, K), f"K mismatch request {r}: {np.argwhere(gk != K)[:5]}"
        assert np.array_equal(gv, V), f"V mismatch request {r}"


# ------------------------------------------------------------------ synth
def test_device_generator_matches_numpy(torch_cuda):
    torch = torch_cuda
    for (L, H, T, D, dtype, heads) in [(2, 2, 64, 64, "fp16", None), (3, 8, 512, 128, "bf16", (2, 5))]:
        h0, h1 = heads or (0, H)
        for kind in (0, 1):
            buf = torch.empty(L * (h1 - h0) * T * D, dtype=torch.int16, device="cuda")
            synth.gen_item_device(buf.data_ptr(), L, H, T, D, 11, kind, heads=heads, dtype=dtype)
            torch.cuda.synchronize()
            want = synth.gen_item(L, H, T, D, 11, kind, heads=heads, dtype=dtype)
            assert np.array_equal(buf.cpu().numpy().view(np.uint16).reshape(want.shape), want)


# -------------------------------------------------------- packed blobs (a3/a4)
@pytest.mark.parametrize("scheme", list(NAMES))
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_packed_blobs_bitexact_tiny(torch_cuda, scheme, dtype):
    st, ora, lay, h, _ = make_pair(torch_cuda, L=2, H=2, T=64, D=64, n_docs=6, ladder=(scheme,), taus=(),
                                   dtype=dtype)
    for item in range(12):
        s, tier, nbytes = st.item_info(item)
        assert s == NAMES[scheme] and nbytes == lay.item_bytes(s)
        assert np.array_equal(st.export_item(item), ora.blobs[item]), (scheme, item)


@pytest.mark.parametrize("scheme", list(NAMES))
@pytest.mark.parametrize("group,gse", [(32, (3, 4)), (4096 * 2, (2, 5))])
def test_packed_blobs_groups_and_layouts(torch_cuda, scheme, group, gse):
    st, ora, lay, h, _ = make_pair(torch_cuda, L=1, H=2, T=128, D=64, n_docs=3, ladder=(scheme,), taus=(),
                                   group=group, gse=gse)
    for item in range(6):
        assert np.array_equal(st.export_item(item), ora.blobs[item]), (scheme, item)


def test_packed_blobs_full_shape_sampled(torch_cuda):
    """Llama-3-8B item shape (32 x 8 x 512 x 128): every scheme's blob, sampled
    slabs recomputed by the oracle one by one."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D = 32, 8, 512, 128
    lay = ost.Layout(L=L, H=H, T=T, D=D)
    rng = np.random.default_rng(0)
    for scheme in NAMES:
        st = hr.Store(L=L, H=H, D=D, T=T, ladder=(scheme,), taus=(), hbm_budget=2 * lay.item_bytes(NAMES[scheme]) + 4096)
        st.build(1, np.array([3, 1], np.uint64), gpu_source(L, H, T, D, "bf16"))
        for item in (0, 1):
            blob = st.export_item(item)
            src = None
            for (l, hh) in [(0, 0), (31, 7)] + [tuple(x) for x in rng.integers(0, [L, H], (2, 2))]:
                if src is None:
                    src = synth.gen_item(L, H, T, D, 0, item)
                c, m = ost.encode_slab(src[l, hh], NAMES[scheme], lay)
                i = l * H + hh
                cb, mo, mr = lay.code_bytes(NAMES[scheme]), lay.meta_offset(NAMES[scheme]), lay.meta_record(NAMES[scheme])
                assert np.array_equal(blob[i * cb:(i + 1) * cb], c), (scheme, item, l, hh)
                assert np.array_equal(blob[mo + i * mr: mo + (i + 1) * mr], m), (scheme, item, l, hh)
        st.close()


def test_nan_rejected(torch_cuda):
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    st = hr.Store(L=1, H=1, D=64, T=64, ladder=("INT8",), taus=(), hbm_budget=1 << 20)
    k = torch.zeros(64 * 64, dtype=torch.int16, device="cuda")
    v = torch.zeros(64 * 64, dtype=torch.int16, device="cuda")
    v[100] = 0x7FC0
    st.build_begin(1, np.zeros(2, np.uint64))
    st.build_put(0, k, v)
    with pytest.raises(hr.HaragError, match="EINVAL"):
        st.build_end()


NONFINITE = {"bf16": {"nan": 0x7FC0, "+inf": 0x7F80, "-inf": 0xFF80, "max": 0x7F7F, "-max": 0xFF7F},
             "fp16": {"nan": 0x7E00, "+inf": 0x7C00, "-inf": 0xFC00, "max": 0x7BFF, "-max": 0xFBFF}}


@pytest.mark.parametrize("scheme", ["PASS16", "INT8", "INT4", "FP8E4M3", "FP8E5M2", "GSE8", "MXFP8"])
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("value", ["nan", "+inf", "-inf", "max", "-max"])
def test_nonfinite_rejected_every_scheme(torch_cuda, scheme, dtype, value):
    """a NaN or +-Inf anywhere in a chunk's source is rejected at ingestion (HR_EINVAL at build end)
    for every scheme's encoder — the INT4 path detects it through its packed NaN-propagating max / min, the
    others through magnitude patterns; the largest finite values are accepted."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    st = hr.Store(L=1, H=1, D=64, T=64, dtype=dtype, ladder=(scheme,), taus=(), hbm_budget=1 << 22)
    rng = np.random.default_rng(7)
    k = torch.zeros(64 * 64, dtype=torch.int16, device="cuda")
    v = torch.zeros(64 * 64, dtype=torch.int16, device="cuda")
    pos = int(rng.integers(0, 64 * 64))
    (k if pos % 2 else v)[pos] = int(np.int16(np.uint16(NONFINITE[dtype][value])))
    st.build_begin(1, np.zeros(2, np.uint64))
    st.build_put(0, k, v)
    if value in ("max", "-max"):
        st.build_end()
    else:
        with pytest.raises(hr.HaragError, match="EINVAL"):
            st.build_end()
    st.close()


# ------------------------------------------------------ assemble (a6-a8, a1)
@pytest.mark.parametrize("ladder,taus,dtype", [(NORTH, (0.25, 0.25), "fp16"), (PAPER, (0.1, 0.1, 0.1), "bf16"),
                                               (PAPER, (0.25, 0.25, 0.25), "fp16")])
def test_assemble_tiny_all_hbm(torch_cuda, ladder, taus, dtype):
    """BASELINE config 0: 16 chunks x 64 tokens, 2 layers, 2 KV heads, head_dim 64, top-k 4."""
    st, ora, lay, h, _ = make_pair(torch_cuda, L=2, H=2, T=64, D=64, n_docs=16, ladder=ladder, taus=taus,
                                   dtype=dtype)
    reqs = synth.gen_requests(16, 64, 4, 1.1, seed=1)
    check_requests(torch_cuda, st, ora, lay, reqs)


def test_assemble_tiny_tiered(torch_cuda):
    """HBM + pinned + pageable tiers (eager placement by bytes) on the tiny config:
    placement equals the oracle's and every output is bit-exact."""
    torch = torch_cuda
    st, ora, lay, h, sizes = make_pair(torch, L=2, H=2, T=64, D=64, n_docs=16, ladder=NORTH, taus=(0.25, 0.25),
                                       dtype="fp16", hbm_items=8, pin_items=8)
    hb = sum(sizes[i] for i in hotness.rank_items(h)[:8])
    pb = sum(sizes[i] for i in hotness.rank_items(h)[8:16])
    want = placement.eager_tiers(h, sizes, hb, pb)
    names = {0: placement.GPU, 1: placement.PIN, 2: placement.PAGE}
    got = [names[st.item_info(i)[1]] for i in range(32)]
    assert got == want
    reqs = synth.gen_requests(16, 64, 4, 1.1, seed=1)
    check_requests(torch, st, ora, lay, reqs)
    s = st.stats()
    assert sum(s["hits"]) == 64 * 4 * 2 and s["hits"][1] > 0 and s["hits"][2] > 0


def test_assemble_pinned_backing_and_ragged(torch_cuda):
    """Pinned backing (config-3 style), ragged slab (T*D = 17408 = 2 tiles + 1024)."""
    st, ora, lay, h, _ = make_pair(torch_cuda, L=2, H=2, T=136, D=128, n_docs=10, ladder=PAPER,
                                   taus=(0.2, 0.2, 0.2), hbm_items=6, backing_pinned=True)
    reqs = synth.gen_requests(10, 12, 3, 1.1, seed=2)
    check_requests(torch_cuda, st, ora, lay, reqs)


def test_assemble_small_slab_and_group32(torch_cuda):
    st, ora, lay, h, _ = make_pair(torch_cuda, L=3, H=4, T=100, D=64, n_docs=8, ladder=("INT4", "INT8", "GSE8"),
                                   taus=(0.3, 0.3), group=32, gse=(3, 4))
    reqs = synth.gen_requests(8, 10, 5, 1.1, seed=3)
    check_requests(torch_cuda, st, ora, lay, reqs)


@pytest.mark.parametrize("world", [2, 4])
def test_head_sharded_equals_oracle(torch_cuda, world):
    """KV-head sharding: each rank's store assembles exactly its
    heads of the unsharded oracle result."""
    reqs = synth.gen_requests(12, 6, 4, 1.1, seed=4)
    full = None
    for rank in range(world):
        st, ora, lay, h, _ = make_pair(torch_cuda, L=2, H=4, T=64, D=64, n_docs=12, ladder=PAPER,
                                       taus=(0.2, 0.2, 0.2), rank=rank, world=world)
        check_requests(torch_cuda, st, ora, lay, reqs)
        if full is None:
            _, fora, flay, _, _ = make_pair(torch_cuda, L=2, H=4, T=64, D=64, n_docs=12, ladder=PAPER,
                                            taus=(0.2, 0.2, 0.2))
            full = [fora.assemble(list(r)) for r in reqs]
        for r, req in enumerate(reqs):
            K, V = ora.assemble(list(req))
            h0, h1 = lay.heads
            assert np.array_equal(K, full[r][0][:, h0:h1]) and np.array_equal(V, full[r][1][:, h0:h1])
        st.close()


def test_assemble_full_shape_sampled(torch_cuda):
    """Llama-3-8B shape, paper ladder, batch of 4 requests x k=10 in the
    launch configuration bench.py times; sampled (l, h) slabs of every output
    checked against the oracle's decode of that slab."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D, n_docs, k = 32, 8, 512, 128, 24, 10
    lay = ost.Layout(L=L, H=H, T=T, D=D)
    prof = synth.gen_requests(n_docs, 200, k, 1.1, seed=9)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in PAPER], (0.1, 0.1, 0.1))
    st = hr.Store(L=L, H=H, D=D, T=T, ladder=PAPER, taus=(0.1, 0.1, 0.1),
                  hbm_budget=sum(lay.item_bytes(s) for s in schemes) + 4096, keep_backing=False)
    st.build(n_docs, h, gpu_source(L, H, T, D, "bf16"))
    reqs = synth.gen_requests(n_docs, 4, k, 1.1, seed=1)
    ko, vo = alloc_out(torch, st, 4, k)
    st.assemble(reqs, ko, vo)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    for r in range(4):
        gk = ko[r].view(L, H, k * T, D)
        gv = vo[r].view(L, H, k * T, D)
        for j in rng.choice(k, 3, replace=False):
            doc = int(reqs[r, j])
            for kind, g in ((0, gk), (1, gv)):
                item = 2 * doc + kind
                src = synth.gen_item(L, H, T, D, doc, kind)
                for (l, hh) in [(0, 0), (L - 1, H - 1), tuple(rng.integers(0, [L, H]))]:
                    c, m = ost.encode_slab(src[l, hh], schemes[item], lay)
                    want = ost.decode_slab(c, m, schemes[item], lay)
                    got = g[l, hh, j * T:(j + 1) * T].cpu().numpy().view(np.uint16).reshape(-1)
                    assert np.array_equal(got, want), (r, j, kind, l, hh)


# ------------------------------------------------------------- hotness / epochs
def test_hotness_delta_counts_and_replace(torch_cuda):
    torch = torch_cuda
    st, ora, lay, h, sizes = make_pair(torch, L=2, H=2, T=64, D=64, n_docs=16, ladder=NORTH, taus=(0.25, 0.25),
                                       dtype="fp16", hbm_items=6, pin_items=6, decay_shift=1)
    hb = sum(sizes[i] for i in hotness.rank_items(h)[:6])
    pb = sum(sizes[i] for i in hotness.rank_items(h)[6:12])
    hcur = h.astype(np.int64)
    for epoch in range(4):
        reqs = synth.gen_requests(16, 40, 4, 1.1, seed=100 + epoch, perm_seed=500 + epoch)
        check_requests(torch, st, ora, lay, reqs)
        delta = st.hotness_delta()
        assert np.array_equal(delta.cpu().numpy(), hotness.count_requests(reqs, 16))
        st.replace()
        hcur = hotness.epoch_update(hcur, hotness.count_requests(reqs, 16), 1)
        want = placement.eager_tiers(hcur, sizes, hb, pb)
        names = {0: placement.GPU, 1: placement.PIN, 2: placement.PAGE}
        assert [names[st.item_info(i)[1]] for i in range(32)] == want, epoch
        assert not st.hotness_delta().any()
    assert st.stats()["migrations_in"] > 0


# --------------------------------------------------------------- error paths
def test_validation_before_any_write(torch_cuda):
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    st, ora, lay, h, _ = make_pair(torch, L=2, H=2, T=64, D=64, n_docs=8, ladder=NORTH, taus=(0.25, 0.25),
                                   dtype="fp16")
    ko, vo = alloc_out(torch, st, 2, 3)
    with pytest.raises(hr.HaragError, match="EINVAL"):
        st.assemble(np.array([[1, 2, 3], [4, 4, 5]]), ko, vo)
    with pytest.raises(hr.HaragError, match="ENOTFOUND"):
        st.assemble(np.array([[1, 2, 3], [4, 8, 5]]), ko, vo)
    torch.cuda.synchronize()
    assert bool((ko[0] == 0x7FFF).all()) and bool((vo[1] == 0x7FFF).all())
    st2 = hr.Store(L=2, H=2, D=64, T=64, ladder=NORTH, taus=(0.25, 0.25), hbm_budget=1 << 20)
    with pytest.raises(hr.HaragError, match="ESTATE"):
        st2.assemble(np.array([[0]]), ko[:1], vo[:1])


def test_put_batch_mixed_tiers_and_validation(torch_cuda):
    """hr_build_put_batch: docs in any order, items of every scheme of the
    north-star ladder and of all tiers (HBM arena, pinned tier, host backing)
    quantised in one launch; blobs equal the oracle's.  Bad batches (repeated
    doc, unknown doc, > 16 docs) fail before any launch."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D, n_docs = 2, 2, 64, 64, 12
    prof = synth.gen_requests(n_docs, 4 * n_docs, 4, 1.1, seed=7)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype="fp16")
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[x] for x in NORTH], (0.25, 0.25))
    sizes = [lay.item_bytes(x) for x in schemes]
    order = hotness.rank_items(h)
    st = hr.Store(L=L, H=H, D=D, T=T, dtype="fp16", ladder=NORTH, taus=(0.25, 0.25),
                  hbm_budget=sum(sizes[i] for i in order[:6]), pin_budget=sum(sizes[i] for i in order[6:10]))
    src = [(torch.from_numpy(synth.gen_item(L, H, T, D, d, 0, dtype="fp16").view(np.int16).reshape(-1).copy()).cuda(),
            torch.from_numpy(synth.gen_item(L, H, T, D, d, 1, dtype="fp16").view(np.int16).reshape(-1).copy()).cuda())
           for d in range(n_docs)]
    st.build_begin(n_docs, h)
    with pytest.raises(hr.HaragError, match="EINVAL"):
        st.build_put_batch([1, 1], [src[1][0]] * 2, [src[1][1]] * 2)
    with pytest.raises(hr.HaragError, match="ENOTFOUND"):
        st.build_put_batch([0, n_docs], [src[0][0]] * 2, [src[0][1]] * 2)
    with pytest.raises(hr.HaragError, match="EINVAL"):
        st.build_put_batch(list(range(17)), [src[0][0]] * 17, [src[0][1]] * 17)
    perm = [7, 3, 11, 0, 5, 9, 1]
    st.build_put_batch(perm, [src[d][0] for d in perm], [src[d][1] for d in perm])
    rest = [d for d in range(n_docs) if d not in perm]
    st.build_put_batch(rest, [src[d][0] for d in rest], [src[d][1] for d in rest])
    st.build_end()
    ora = ost.OracleStore(lay, [NAMES[x] for x in NORTH], (0.25, 0.25))
    ora.build(n_docs, h, lambda d, k: synth.gen_item(L, H, T, D, d, k, dtype="fp16"))
    tiers = set()
    for item in range(2 * n_docs):
        s_, tier, _ = st.item_info(item)
        tiers.add(tier)
        assert np.array_equal(st.export_item(item), ora.blobs[item]), item
    assert len(tiers) == 3


# ------------------------------------------------- demand mode (paper-literal Alg. 2)
@pytest.mark.parametrize("backing_pinned", [False, True])
def test_demand_mode_matches_oracle_alg2(torch_cuda, backing_pinned):
    """demand_mode = 1: queues start empty; every access takes one Alg. 2 branch
     with inclusive promotion and LRU (R16).  Per-tier hit counts and
    the queue contents after every call equal the oracle's Alg2 run on the same
    access order, and every output stays bit-exact."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D, n_docs = 2, 2, 64, 64, 16
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype="fp16")
    prof = synth.gen_requests(n_docs, 64, 4, 1.1, seed=7)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    ladder, taus = NORTH, (0.25, 0.25)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in ladder], taus)
    sizes = [lay.item_bytes(s) for s in schemes]
    order = hotness.rank_items(h)
    hb = sum(sizes[i] for i in order[:10]) - 1      # capacity slightly below the list: LRU fires
    pb = 0 if backing_pinned else sum(sizes[i] for i in order[10:16])
    st = hr.Store(L=L, H=H, D=D, T=T, dtype="fp16", ladder=ladder, taus=taus, hbm_budget=hb, pin_budget=pb,
                  backing_pinned=backing_pinned, demand_mode=True)
    st.build(n_docs, h, gpu_source(L, H, T, D, "fp16"))
    ora = ost.OracleStore(lay, [NAMES[s] for s in ladder], taus)
    ora.build(n_docs, h, lambda d, k: synth.gen_item(L, H, T, D, d, k, dtype="fp16"))
    gl, pl, rest = placement.lists_by_bytes(order, sizes, hb, pb)
    alg = placement.Alg2(gl, pl, rest, (hb, pb, 0), sizes)
    names = {placement.GPU: 0, placement.PIN: 1, placement.PAGE: 2, placement.DISK: 2}
    want_hits = [0, 0, 0]
    for call in range(6):
        reqs = synth.gen_requests(n_docs, 5, 4, 1.1, seed=40 + call)
        check_requests(torch, st, ora, lay, reqs)
        for req in reqs:
            for doc in req:
                for kind in (0, 1):
                    want_hits[names[alg.access(2 * int(doc) + kind)[0]]] += 1
        assert st.stats()["hits"] == want_hits, call
        gpu_q = set(alg.resident(placement.GPU))
        pin_q = set(alg.resident(placement.PIN))
        got = [st.item_info(i)[1] for i in range(2 * n_docs)]
        assert {i for i in range(2 * n_docs) if got[i] == 0} == gpu_q, call
        assert {i for i in range(2 * n_docs) if got[i] == 1} == pin_q - gpu_q, call
        # physical residency follows queueGPU: the HBM arena holds exactly its items (no leaked or
        # lagging arena blocks) and nothing else
        res = [st.item_residency(i) for i in range(2 * n_docs)]
        assert {i for i in range(2 * n_docs) if res[i] & hr.R_HBM} == gpu_q, call
        assert st.stats()["hbm_used"] == sum((sizes[i] + 255) // 256 * 256 for i in gpu_q), call
    s = st.stats()
    assert s["hbm_used"] <= hb and s["migrations_in"] > 0 and s["failed_promotions"] == 0


@pytest.mark.parametrize("page_items", [0, 4])
def test_demand_mode_four_tiers_matches_oracle(torch_cuda, tmp_path, page_items):
    """Disk-backed store in demand mode: all four lists and three queues of
    Alg. 2 — a PAGE_LIST hit serves the pageable cache, a miss
    reads the file and fills every queue its list names (R16, R26).  Per-tier
    hit counts (DISK included) and queue contents match the oracle Alg2 after
    every call; outputs stay bit-exact."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    st, ora, lay, h, sizes = make_pair(torch, L=2, H=2, T=64, D=64, n_docs=16, ladder=NORTH, taus=(0.25, 0.25),
                                       dtype="fp16")
    path = str(tmp_path / "store4.hr")
    st.save(path)
    st.close()
    order = hotness.rank_items(h)
    hb = sum(sizes[i] for i in order[:8]) - 1
    pb = sum(sizes[i] for i in order[8:12])
    gb = sum(sizes[i] for i in order[12:12 + page_items])
    ld = hr.Store(L=2, H=2, D=64, T=64, dtype="fp16", hbm_budget=hb, pin_budget=pb, page_budget=gb,
                  disk_backing=True, demand_mode=True, keep_backing=False)
    ld.build_from_file(path)
    gl, pl, al, dl = placement.lists_by_bytes4(order, sizes, hb, pb, gb)
    alg = placement.Alg2(gl, pl, al, (hb, pb, gb), sizes)
    idx = {placement.GPU: 0, placement.PIN: 1, placement.PAGE: 2, placement.DISK: 3}
    want = [0, 0, 0, 0]
    for call in range(6):
        reqs = synth.gen_requests(16, 5, 4, 1.1, seed=80 + call)
        check_requests(torch, ld, ora, lay, reqs)
        for req in reqs:
            for doc in req:
                for kind in (0, 1):
                    want[idx[alg.access(2 * int(doc) + kind)[0]]] += 1
        s = ld.stats()
        assert s["hits"] == want[:3] and s["hits_disk"] == want[3], call
        q = [set(alg.resident(t)) for t in (placement.GPU, placement.PIN, placement.PAGE)]
        got = [ld.item_info(i)[1] for i in range(32)]
        exp = [0 if i in q[0] else 1 if i in q[1] else 2 if i in q[2] else 3 for i in range(32)]
        assert got == exp, call
        res = [ld.item_residency(i) for i in range(32)]
        assert {i for i in range(32) if res[i] & hr.R_HBM} == q[0], call
        assert all(r & hr.R_FILE for r in res)
    assert want[3] > 0 and (page_items == 0 or want[2] > 0)
    ld.close()


# ------------------------------------------- BASELINE configs 2-4 at full shape
def _sampled_check(torch, st, reqs, outs, lay, schemes, rng, n_slabs=2, src_heads=None):
    """Oracle decode of sampled (request, slot, kind, layer, head) slabs, one by one."""
    L, Hl, T, D = lay.L, lay.Hl, lay.T, lay.D
    k = reqs.shape[1]
    for r in range(len(reqs)):
        for j in rng.choice(k, min(2, k), replace=False):
            doc = int(reqs[r, j])
            for kind in (0, 1):
                item = 2 * doc + kind
                g = outs[kind][r].view(L, Hl, k * T, D)
                for _ in range(n_slabs):
                    l, hh = int(rng.integers(L)), int(rng.integers(Hl))
                    h_glob = lay.heads[0] + hh
                    x = synth.gen_item(L, lay.H, T, D, doc, kind, heads=(h_glob, h_glob + 1))[l, 0]
                    c, m = ost.encode_slab(x, schemes[item], lay)
                    want = ost.decode_slab(c, m, schemes[item], lay)
                    got = g[l, hh, j * T:(j + 1) * T].cpu().numpy().view(np.uint16).reshape(-1)
                    assert np.array_equal(got, want), (r, j, kind, l, hh)


def test_config2_llama2_mha_tiered_sampled(torch_cuda):
    """BASELINE config 2: Llama-2-7B MHA KV shape (32 layers x 32 heads x 128),
    hot items in HBM, cold in pinned host DRAM, batch of requests; sampled slabs."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D, n_docs, k, B = 32, 32, 512, 128, 14, 4, 4
    lay = ost.Layout(L=L, H=H, T=T, D=D)
    prof = synth.gen_requests(n_docs, 80, k, 1.1, seed=9)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in PAPER], (0.1, 0.1, 0.1))
    order = hotness.rank_items(h)
    hb = sum(lay.item_bytes(schemes[i]) for i in order[:8])
    st = hr.Store(L=L, H=H, D=D, T=T, ladder=PAPER, taus=(0.1, 0.1, 0.1), hbm_budget=hb,
                  backing_pinned=True, keep_backing=True)
    st.build(n_docs, h, gpu_source(L, H, T, D, "bf16"))
    tiers = [st.item_info(i)[1] for i in range(2 * n_docs)]
    assert tiers.count(0) == 8 and tiers.count(1) == 2 * n_docs - 8
    reqs = synth.gen_requests(n_docs, B, k, 1.1, seed=3)
    ko, vo = alloc_out(torch, st, B, k)
    st.assemble(reqs, ko, vo)
    torch.cuda.synchronize()
    assert st.stats()["hits"][1] > 0
    _sampled_check(torch, st, reqs, (ko, vo), lay, schemes, np.random.default_rng(1))


@pytest.mark.parametrize("world", [2, 8])
def test_config3_llama3_70b_sharded_sampled(torch_cuda, world):
    """BASELINE config 3: Llama-3-70B KV shape (80 layers x 8 KV heads), KV-head
    sharded across `world` ranks (stores built one rank at a time on this GPU)."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D, n_docs, k, B = 80, 8, 512, 128, 10, 4, 2
    prof = synth.gen_requests(n_docs, 60, k, 1.1, seed=11)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in NORTH], (0.2, 0.3))
    reqs = synth.gen_requests(n_docs, B, k, 1.1, seed=5)
    for rank in (0, world - 1):
        lay = ost.Layout(L=L, H=H, T=T, D=D, rank=rank, world=world)
        st = hr.Store(L=L, H=H, D=D, T=T, ladder=NORTH, taus=(0.2, 0.3), rank=rank, world=world,
                      hbm_budget=sum(lay.item_bytes(s) for s in schemes) + 4096, keep_backing=False)
        st.build(n_docs, h, gpu_source(L, H, T, D, "bf16"))
        ko, vo = alloc_out(torch, st, B, k)
        st.assemble(reqs, ko, vo)
        torch.cuda.synchronize()
        _sampled_check(torch, st, reqs, (ko, vo), lay, schemes, np.random.default_rng(rank))
        # request q is counted by rank q mod world only
        d = st.hotness_delta().cpu().numpy()
        assert np.array_equal(d, hotness.count_requests(reqs, n_docs, rank, world))
        st.close()


def test_config4_hotness_drift_replacement(torch_cuda):
    """BASELINE config 4 (scaled): re-placement under shifting Zipf skew
    (s = 0.6 -> 0.8 -> 1.0 -> 1.2 -> 0.6, fresh permutation per phase), per-rank
    view of 8-way head sharding of the Llama-3-8B shape (1 KV head per rank),
    decay_shift 1, an epoch per phase: placement after every epoch equals the
    oracle's, and assembled slabs stay bit-exact across migrations."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    L, H, T, D, n_docs, k, world = 32, 8, 512, 128, 40, 8, 8
    lay = ost.Layout(L=L, H=H, T=T, D=D, rank=0, world=world)
    prof = synth.gen_requests(n_docs, 100, k, 1.1, seed=12)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in PAPER], (0.1, 0.1, 0.1))
    sizes = [lay.item_bytes(s) for s in schemes]
    order = hotness.rank_items(h)
    hb = sum(sizes[i] for i in order[:20])
    pb = sum(sizes[i] for i in order[20:40])
    st = hr.Store(L=L, H=H, D=D, T=T, ladder=PAPER, taus=(0.1, 0.1, 0.1), rank=0, world=world,
                  hbm_budget=hb, pin_budget=pb, keep_backing=True, decay_shift=1)
    st.build(n_docs, h, gpu_source(L, H, T, D, "bf16"))
    hcur = h.astype(np.int64)
    names = {0: placement.GPU, 1: placement.PIN, 2: placement.PAGE}
    rng = np.random.default_rng(4)
    for phase, s in enumerate((0.6, 0.8, 1.0, 1.2, 0.6)):
        reqs = synth.gen_requests(n_docs, 32, k, s, seed=200 + phase, perm_seed=300 + phase)
        ko, vo = alloc_out(torch, st, len(reqs), k)
        st.assemble(reqs, ko, vo)
        torch.cuda.synchronize()
        _sampled_check(torch, st, reqs[:3], (ko[:3], vo[:3]), lay, schemes, rng, n_slabs=1)
        # the all-reduce of the 8 ranks' deltas equals the count of every request
        full = hotness.count_requests(reqs, n_docs)
        st.hotness_delta().copy_(torch.from_numpy(full).cuda())
        st.replace()
        hcur = hotness.epoch_update(hcur, full, 1)
        want = placement.eager_tiers(hcur, sizes, hb, pb)
        assert [names[st.item_info(i)[1]] for i in range(2 * n_docs)] == want, phase
    assert st.stats()["migrations_in"] > 0


@pytest.mark.parametrize("scheme", ["INT8", "INT4"])
def test_quantize_exact_ties(torch_cuda, scheme):
    """Groups whose quotients x/s land exactly on half-integers (ties to even)
    and within a few ulps of them: the GPU's division-free fast path must fall
    back to the IEEE quotient there (R3) — packed blobs equal the oracle's."""
    import paper_2510_20878_b200 as hr
    from oracle import numerics
    torch = torch_cuda
    L, H, T, D = 1, 1, 64, 128
    rng = np.random.default_rng(3)
    vals = np.empty((T, D), np.float32)
    for t in range(T):
        j = int(rng.integers(-20, 10))
        top = 127 if scheme == "INT8" else 15
        k = rng.integers(0, top, D).astype(np.float32)
        row = (k + np.float32(0.5)) * np.float32(2.0 ** j)
        if t % 2:   # nudge by a few ulps around the tie
            row = np.nextafter(row, np.float32(np.inf) * rng.choice([-1, 1], D)).astype(np.float32)
        row[0] = np.float32(top * 2.0 ** j)          # the group's max |x| (INT8) / max (INT4)
        if scheme == "INT4":
            row[1] = np.float32(0.0)                  # min = 0 -> s = 2^j exactly
        if scheme == "INT8" and t % 3 == 0:
            row = -row
        vals[t] = row
    bits = numerics.f32_to_bf16(vals).reshape(L, H, T, D)
    lay = ost.Layout(L=L, H=H, T=T, D=D)
    want = ost.encode_item(bits, NAMES[scheme], lay)
    st = hr.Store(L=L, H=H, D=D, T=T, ladder=(scheme,), taus=(), hbm_budget=1 << 20)
    src = torch.from_numpy(bits.view(np.int16).reshape(-1).copy()).cuda()
    st.build_begin(1, np.zeros(2, np.uint64))
    st.build_put(0, src, src)
    st.build_end()
    assert np.array_equal(st.export_item(0), want)


def _edge_source(dtype, rng, L=2, H=2, T=64, D=128):
    """Slabs of special values: signed zeros, subnormals, the smallest normal,
    the largest finite value, FP8 saturation neighbours, all-tiny slabs,
    all-zero groups, and exponent ranges wider than any GSE-8 array."""
    n = T * D
    if dtype == "bf16":
        special = [0x0000, 0x8000, 0x0001, 0x807F, 0x0080, 0x8080, 0x7F7F, 0xFF7F, 0x43E0, 0x43E1, 0xC3E1,
                   0x4780, 0x477F, 0x3F80, 0x3F81, 0x0100, 0x2000, 0x6000]
        rand = lambda k: rng.integers(0, 0x7F80, k).astype(np.uint16) | (rng.integers(0, 2, k) << 15).astype(np.uint16)
        tiny = lambda k: rng.integers(0, 0x0080, k).astype(np.uint16) | (rng.integers(0, 2, k) << 15).astype(np.uint16)
        huge = lambda k: rng.integers(0x7B00, 0x7F80, k).astype(np.uint16)
    else:
        special = [0x0000, 0x8000, 0x0001, 0x83FF, 0x0400, 0x7BFF, 0xFBFF, 0x5F00, 0x5F08, 0x3C00, 0x3C01, 0x7800]
        rand = lambda k: rng.integers(0, 0x7C00, k).astype(np.uint16) | (rng.integers(0, 2, k) << 15).astype(np.uint16)
        tiny = lambda k: rng.integers(0, 0x0400, k).astype(np.uint16)
        huge = lambda k: rng.integers(0x7000, 0x7C00, k).astype(np.uint16)
    slabs = []
    a = rand(n)
    a[: len(special)] = special
    a[1024:1152] = 0                                   # an all-zero group (INT8/INT4)
    a[2048:2176] = tiny(128)                           # a subnormal-only group
    slabs.append(a)
    slabs.append(np.where(rng.random(n) < 0.5, 0, tiny(n)).astype(np.uint16))     # only zeros/subnormals
    h = huge(n)
    h[::7] = rand(len(h[::7]))
    slabs.append(h)                                    # huge values + a wide exponent range
    slabs.append(np.zeros(n, np.uint16))               # all zero
    return np.stack(slabs).reshape(L, H, T, D)


@pytest.mark.parametrize("scheme", list(NAMES))
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_edge_values_bitexact(torch_cuda, scheme, dtype):
    """Degenerate inputs for every scheme: blobs and decoded outputs equal the oracle's."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    rng = np.random.default_rng(17)
    L, H, T, D = 2, 2, 64, 128
    k_bits = _edge_source(dtype, rng)
    v_bits = _edge_source(dtype, rng)[::-1].copy()
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype=dtype)
    st = hr.Store(L=L, H=H, D=D, T=T, dtype=dtype, ladder=(scheme,), taus=(), hbm_budget=1 << 22)
    ks = torch.from_numpy(k_bits.view(np.int16).reshape(-1).copy()).cuda()
    vs = torch.from_numpy(v_bits.view(np.int16).reshape(-1).copy()).cuda()
    st.build_begin(1, np.zeros(2, np.uint64))
    st.build_put(0, ks, vs)
    st.build_end()
    for item, bits in ((0, k_bits), (1, v_bits)):
        want_blob = ost.encode_item(bits, NAMES[scheme], lay)
        assert np.array_equal(st.export_item(item), want_blob), (scheme, dtype, item)
    ko, vo = alloc_out(torch, st, 1, 1)
    st.assemble(np.array([[0]]), ko, vo)
    torch.cuda.synchronize()
    for out, item in ((ko[0], 0), (vo[0], 1)):
        want = ost.decode_item(st.export_item(item), NAMES[scheme], lay)
        got = out.cpu().numpy().view(np.uint16).reshape(want.shape)
        assert np.array_equal(got, want), (scheme, dtype, item, np.argwhere(got != want)[:4])


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_int8_scale_all_16bit_values(torch_cuda, dtype):
    """The INT8 scale fl(a/127) is computed without a division (Markstein
    correction); a is a 16-bit source value, so checking every
    finite magnitude covers its whole domain: one group of G = 32 per value
    (value first, zeros after), scales and codes equal the oracle's."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    top = 0x7F7F if dtype == "bf16" else 0x7BFF
    mags = np.arange(0, top + 1, dtype=np.uint32).astype(np.uint16)
    n = mags.size
    pad = (-n) % 8                       # whole 256-element chunks: T*D % 256 == 0
    vals = np.concatenate([mags, np.zeros(pad, np.uint16)])
    groups = np.zeros((vals.size, 32), np.uint16)
    groups[:, 0] = vals
    groups[::3, 0] |= 0x8000             # negative maxima too
    groups[:, 5] = vals >> 1              # a smaller magnitude in the group
    L, H, D = 1, 1, 128
    T = groups.size // D
    bits = groups.reshape(L, H, T, D)
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype=dtype, group=32)
    want = ost.encode_item(bits, ost.INT8, lay)
    st = hr.Store(L=L, H=H, D=D, T=T, dtype=dtype, group=32, ladder=("INT8",), taus=(),
                  hbm_budget=2 * lay.item_bytes(ost.INT8) + (1 << 20))
    src = torch.from_numpy(bits.view(np.int16).reshape(-1).copy()).cuda()
    st.build_begin(1, np.zeros(2, np.uint64))
    st.build_put(0, src, src)
    st.build_end()
    got = st.export_item(0)
    mo = lay.meta_offset(ost.INT8)
    assert np.array_equal(got[mo:mo + 4 * T * D // 32], want[mo:mo + 4 * T * D // 32]), "scales"
    assert np.array_equal(got, want)


def test_markstein_division_exhaustive(torch_cuda):
    """The INT8 / INT4 quantizers compute fl(x/s) without a division
    (Markstein's FMA correction).  tests/csrc/markstein_check.cu
    compares INT8 with IEEE division for every pair of 16-bit values (a, x),
    |x| <= a, bf16 and fp16 (2.07e9 pairs), and INT4's two-correction variant
    on 2^36 sampled (x, mn, mx) triples per dtype, half of them steered onto
    quantisation ties: zero mismatches required."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "csrc", "markstein_check")
    assert os.path.exists(exe), "build() compiles tests/csrc/markstein_check"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "mismatches 0" in r.stdout.splitlines()[-1], r.stdout


# ----------------------------------------------------- persistence and the DISK tier
@pytest.mark.parametrize("disk_backing,demand,page", [(False, False, 0), (True, False, 0), (True, True, 0),
                                                       (True, False, 3), (True, True, 3)])
def test_save_load_and_disk_tier(torch_cuda, tmp_path, disk_backing, demand, page):
    """hr_store_save / hr_build_from_file: compress once, load many.
    The loaded store keeps the saved schemes, places by its own budgets, and
    with disk_backing = 1 serves cold items from the file on every miss (the
    DISK tier); outputs stay bit-exact, re-placement too."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    st, ora, lay, h, sizes = make_pair(torch, L=2, H=2, T=64, D=64, n_docs=16, ladder=NORTH, taus=(0.25, 0.25),
                                       dtype="fp16")
    path = str(tmp_path / "store.hr")
    st.save(path)
    order = hotness.rank_items(h)
    hb = sum(sizes[i] for i in order[:6])
    pb = sum(sizes[i] for i in order[6:10])
    gb = sum(sizes[i] for i in order[10:10 + page])     # PAGE_LIST cache of the disk-backed store (R26)
    ld = hr.Store(L=2, H=2, D=64, T=64, dtype="fp16", ladder=("INT8",), taus=(), hbm_budget=hb, pin_budget=pb,
                  disk_backing=disk_backing, demand_mode=demand, keep_backing=not disk_backing, page_budget=gb)
    ld.build_from_file(path)
    for item in range(32):
        assert ld.item_info(item)[0] == st.item_info(item)[0]          # saved schemes, not the new ladder
        assert np.array_equal(ld.export_item(item), ora.blobs[item])
    if not demand:
        want = placement.eager_tiers(h, sizes, hb, pb, page_budget=gb if disk_backing else None)
        names = {0: placement.GPU, 1: placement.PIN, 2: placement.PAGE, 3: placement.DISK}
        assert [names[ld.item_info(i)[1]] for i in range(32)] == want
    for epoch in range(3):
        reqs = synth.gen_requests(16, 24, 4, 1.1, seed=60 + epoch, perm_seed=70 + epoch)
        check_requests(torch, ld, ora, lay, reqs)
        ld.replace()
    s = ld.stats()
    assert s["hits"][2] > 0 or s["hits"][1] > 0
    if disk_backing:
        assert s["hits_disk"] > 0
    ld.close()
    with open(path, "r+b") as f:   # corrupt the magic
        f.write(b"XXXX")
    bad = hr.Store(L=2, H=2, D=64, T=64, dtype="fp16", hbm_budget=hb)
    with pytest.raises(hr.HaragError, match="ECORRUPT"):
        bad.build_from_file(path)
    other = hr.Store(L=2, H=2, D=128, T=64, dtype="fp16", hbm_budget=hb)
    st.save(path)
    with pytest.raises(hr.HaragError, match="EINVAL"):
        other.build_from_file(path)


def test_refused_replace_leaves_epoch_state(torch_cuda):
    """hr_replace that cannot migrate (keep_backing = 0 and the lists move) returns HR_ESTATE and
    leaves hotness, rank order and the accumulated delta exactly as they were."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    st, ora, lay, h, sizes = make_pair(torch, L=2, H=2, T=64, D=64, n_docs=8, ladder=NORTH, taus=(0.25, 0.25),
                                       dtype="fp16", hbm_items=4, keep_backing=False)
    ranks = [st.item_rank(i) for i in range(16)]
    cold = [i for i in range(16) if ranks[i] >= 8]
    delta = np.zeros(16, np.int64)
    delta[cold] = 1000                                   # the cold items would take over the HBM set
    st.hotness_delta().copy_(torch.from_numpy(delta).cuda())
    with pytest.raises(hr.HaragError, match="ESTATE"):
        st.replace()
    assert [st.item_rank(i) for i in range(16)] == ranks
    assert np.array_equal(st.hotness_delta().cpu().numpy(), delta)
    reqs = synth.gen_requests(8, 6, 3, 1.1, seed=9)
    check_requests(torch, st, ora, lay, reqs)


def test_tail_balanced_launches_reuse_their_counters(torch_cuda):
    """Assemble's tail balancing claims the last quarter of every launch's tiles through a per-launch
    counter (64 slots per store, zeroed by the launch's last producer): 70 consecutive launches (every slot
    reused) on two alternating streams each produce every element of every request exactly as the oracle."""
    torch = torch_cuda
    # 8 requests x 4 docs x 2 items x 16 slabs x 1 tile = 1,024 tiles >= 4 x 148 CTAs: the dynamic tail is on
    st, ora, lay, h, _ = make_pair(torch, L=4, H=4, T=128, D=64, n_docs=12, ladder=PAPER, taus=(0.2, 0.2, 0.2))
    reqs = synth.gen_requests(12, 8, 4, 1.1, seed=21)
    want = [ora.assemble(list(r)) for r in reqs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ko, vo = alloc_out(torch, st, len(reqs), 4)
    for it in range(70):
        s = streams[it % 2]
        s.wait_stream(streams[(it + 1) % 2])  # the outputs are reused: order the launches
        for t in ko + vo:
            t.record_stream(s)
        with torch.cuda.stream(s):
            for t in ko + vo:
                t.fill_(0x7FFF)
        st.assemble(reqs, ko, vo, stream=s)
        if it % 23 == 0 or it == 69:
            s.synchronize()
            for r, (K, V) in enumerate(want):
                assert np.array_equal(ko[r].cpu().numpy().view(np.uint16).reshape(K.shape), K), (it, r)
                assert np.array_equal(vo[r].cpu().numpy().view(np.uint16).reshape(V.shape), V), (it, r)
    st.close()


def test_metrics_jsonl_per_call(torch_cuda, tmp_path, monkeypatch):
    """HARAG_METRICS_JSONL (SURVEY §5 metrics): one JSON line per hr_assemble_kv call whose counters add up
    to the call — every item of every request counted once in a tier, KV bytes = 2 x n_req x kv_bytes(k)."""
    import json
    path = tmp_path / "m.jsonl"
    monkeypatch.setenv("HARAG_METRICS_JSONL", str(path))
    torch = torch_cuda
    st, ora, lay, h, _ = make_pair(torch, L=2, H=2, T=64, D=64, n_docs=8, ladder=PAPER, taus=(0.2, 0.2, 0.2),
                                   hbm_items=6)
    reqs = [synth.gen_requests(8, n, 3, 1.1, seed=30 + n) for n in (1, 2, 4)]
    for r in reqs:
        ko, vo = alloc_out(torch, st, len(r), 3)
        st.assemble(r, ko, vo)
    torch.cuda.synchronize()
    st.close()
    lines = [json.loads(x) for x in path.read_text().splitlines()]
    assert [x["call"] for x in lines] == [0, 1, 2]
    for x, r in zip(lines, reqs):
        assert x["n_req"] == len(r) and x["k"] == 3
        assert sum(x["hits"]) + x["hits_disk"] == 2 * len(r) * 3
        assert x["bytes_out"] == 2 * len(r) * st_kv_bytes(lay, 3)
        assert x["host_us"] > 0


def st_kv_bytes(lay, k):
    return 2 * lay.L * lay.Hl * k * lay.T * lay.D
