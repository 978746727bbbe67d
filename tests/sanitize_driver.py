"""Small workload that launches every sm_100a kernel of libharag on tiny shapes, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck; tools/sanitize.sh).  Test
infrastructure (it calls the oracle), kept under tests/ but not collected by pytest.

Kernels exercised: quantize_batch_kernel (INT8 / INT4 TMA ring, GSE-8 range + encode passes),
quant_tile_kernel (PASS16 / FP8), gse_slab_kernel (4-CTA cluster, DSMEM), quant_biggroup_kernel
(G = T*D), assemble_kv_kernel (HBM-resident launch A, streamed launch B from pinned and pageable
tiers, ragged slabs, PASS16 bulk write-back), attend_kernel (tcgen05 / TMEM, D = 64 and 128),
exponent_hist_kernel and the error kernels.  Every output is also checked against the oracle, so
a clean sanitizer log is a log of a correct run.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_20878_b200 as hr  # noqa: E402
import synth  # noqa: E402
from oracle import attention, hotness  # noqa: E402
from oracle import store as ost  # noqa: E402

# HARAG_SAN_NO_PASS16=1: ladders without PASS16 (whose tiles the kernels write with the bulk-copy engine,
# cp.async.bulk shared -> global, which initcheck does not see as initialising device memory)
NO_PASS16 = bool(os.environ.get("HARAG_SAN_NO_PASS16"))
NAMES = {"PASS16": ost.PASS16, "INT8": ost.INT8, "FP8E4M3": ost.FP8E4M3, "FP8E5M2": ost.FP8E5M2,
         "GSE8": ost.GSE8, "INT4": ost.INT4, "MXFP8": ost.MXFP8}


def make(L, H, T, D, n_docs, ladder, taus, dtype="bf16", group=0, hbm_items=None, pin_items=0, pinned=False):
    if NO_PASS16:
        ladder = tuple("INT8" if s == "PASS16" else s for s in ladder)
    prof = synth.gen_requests(n_docs, 4 * n_docs, min(4, n_docs), 1.1, seed=7)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype=dtype, group=group)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in ladder], taus)
    sizes = [lay.item_bytes(s) for s in schemes]
    order = hotness.rank_items(h)
    hb = sum(sizes) + 4096 if hbm_items is None else sum(sizes[i] for i in order[:hbm_items])
    pb = 0 if hbm_items is None else sum(sizes[i] for i in order[hbm_items:hbm_items + pin_items])
    st = hr.Store(L=L, H=H, D=D, T=T, dtype=dtype, group=group, ladder=ladder, taus=taus, hbm_budget=hb,
                  pin_budget=pb, backing_pinned=pinned, keep_backing=True)

    def src(doc, kp, vp, stream):
        synth.gen_item_device(kp, L, H, T, D, doc, 0, dtype=dtype, stream=stream)
        synth.gen_item_device(vp, L, H, T, D, doc, 1, dtype=dtype, stream=stream)

    st.build(n_docs, h, src)
    ora = ost.OracleStore(lay, [NAMES[s] for s in ladder], taus)
    ora.build(n_docs, h, lambda d, k: synth.gen_item(L, H, T, D, d, k, dtype=dtype))
    return st, ora, lay


def check_assemble(st, ora, reqs):
    nb = st.kv_bytes(reqs.shape[1])
    ko = [torch.empty(nb // 2, dtype=torch.int16, device="cuda") for _ in reqs]
    vo = [torch.empty(nb // 2, dtype=torch.int16, device="cuda") for _ in reqs]
    st.assemble(reqs, ko, vo)
    torch.cuda.synchronize()
    for r, req in enumerate(reqs):
        K, V = ora.assemble(list(req))
        assert np.array_equal(ko[r].cpu().numpy().view(np.uint16).reshape(K.shape), K)
        assert np.array_equal(vo[r].cpu().numpy().view(np.uint16).reshape(V.shape), V)


def main():
    torch.cuda.set_device(0)
    n = 0
    # quantize (every scheme, both dtypes) + HBM-resident assemble
    for dtype in ("bf16", "fp16"):
        for ladder, taus in ((("PASS16", "INT8", "INT4"), (0.25, 0.25)),
                             (("INT8", "FP8E4M3", "FP8E5M2", "GSE8"), (0.2, 0.2, 0.2))):
            st, ora, lay = make(2, 2, 64, 64, 8, ladder, taus, dtype=dtype)
            for i in range(16):
                assert np.array_equal(st.export_item(i), ora.blobs[i])
            check_assemble(st, ora, synth.gen_requests(8, 4, 3, 1.1, seed=1))
            st.close()
            n += 1
    # paper-ratio groups (quant_biggroup_kernel) and group 32
    for group in (64 * 64, 32):
        st, ora, lay = make(1, 2, 64, 64, 4, ("INT8", "INT4"), (0.5,), group=group)
        for i in range(8):
            assert np.array_equal(st.export_item(i), ora.blobs[i])
        check_assemble(st, ora, synth.gen_requests(4, 2, 2, 1.1, seed=2))
        st.close()
    # host tiers: pinned tier + pageable backing, and a pinned backing; ragged slab (T*D = 17408)
    st, ora, lay = make(2, 2, 136, 128, 10, ("INT8", "FP8E4M3", "FP8E5M2", "GSE8"), (0.2, 0.2, 0.2),
                        hbm_items=6, pin_items=6)
    check_assemble(st, ora, synth.gen_requests(10, 6, 3, 1.1, seed=3))
    st.replace()
    check_assemble(st, ora, synth.gen_requests(10, 6, 3, 1.1, seed=4))
    st.close()
    st, ora, lay = make(2, 2, 64, 64, 10, ("PASS16", "INT8", "INT4"), (0.25, 0.25), hbm_items=4, pinned=True)
    check_assemble(st, ora, synth.gen_requests(10, 6, 3, 1.1, seed=5))
    st.close()
    # attention consumer (tcgen05 / TMEM)
    for D in (64, 128):
        st, ora, lay = make(2, 2, 128, D, 6, ("INT8", "FP8E4M3", "FP8E5M2", "GSE8"), (0.2, 0.2, 0.2))
        reqs = synth.gen_requests(6, 2, 2, 1.1, seed=6).astype(np.uint32)
        g, n_q = 2, 8
        q = torch.from_numpy(synth.gen_query(2, 2, 2 * g, n_q, D).view(np.int16)).cuda()
        o = torch.empty_like(q)
        lse = torch.empty((2, 2, 2 * g, n_q), dtype=torch.float32, device="cuda")
        st.attend(reqs, q, o, n_q, g, lse=lse)
        torch.cuda.synchronize()
        qb = synth.gen_query(2, 2, 2 * g, n_q, D)
        for r in range(2):
            K, V = ora.assemble(list(reqs[r]))
            O, lse_w = attention.attend_request(qb[r], K, V, g, "bf16")
            got = o[r].view(torch.bfloat16).float().cpu().numpy().astype(np.float64)
            vr = np.abs(ost.numerics.to_f32(V, "bf16")).max()
            assert np.all(np.abs(got - O) <= 2.0 ** -8 * 2 * vr + 2.0 ** -8 * np.abs(O) + 1e-6), D
            assert np.all(np.abs(lse[r].cpu().numpy() - lse_w) <= 2.0 ** -8), D
        st.close()
    # MXFP8 (R31): quantize (tile kernel) + assemble, both dtypes
    for dtype in ("bf16", "fp16"):
        st, ora, lay = make(2, 2, 64, 64, 8, ("MXFP8", "GSE8"), (0.5,), dtype=dtype)
        for i in range(16):
            assert np.array_equal(st.export_item(i), ora.blobs[i])
        check_assemble(st, ora, synth.gen_requests(8, 4, 3, 1.1, seed=7))
        st.close()
        n += 1
    # attention prefill form (R30): chunk keys + the question's own K/V, causal; forced 3 splits (the own
    # tile alone in the last one)
    os.environ["HARAG_ATT_SPLIT"] = "3"
    st, ora, lay = make(2, 2, 64, 128, 6, ("INT8", "FP8E4M3", "FP8E5M2", "GSE8"), (0.2, 0.2, 0.2))
    reqs = synth.gen_requests(6, 2, 2, 1.1, seed=8).astype(np.uint32)
    g, n_q, D = 2, 8, 128
    qb = synth.gen_query(2, 2, 2 * g, n_q, D)
    kob, vob = synth.gen_query(2, 2, 2, n_q, D, seed=91), synth.gen_query(2, 2, 2, n_q, D, seed=92)
    cu = lambda a: torch.from_numpy(a.view(np.int16)).cuda()  # noqa: E731
    q, ko, vo = cu(qb), cu(kob), cu(vob)
    o = torch.empty_like(q)
    lse = torch.empty((2, 2, 2 * g, n_q), dtype=torch.float32, device="cuda")
    st.attend_prefill(reqs, q, ko, vo, o, n_q, g, layers=(0, 2), lse=lse)
    torch.cuda.synchronize()
    for r in range(2):
        K, V = ora.assemble(list(reqs[r]))
        O, lse_w = attention.attend_request(qb[r], K, V, g, "bf16", K_own_bits=kob[r], V_own_bits=vob[r])
        got = o[r].view(torch.bfloat16).float().cpu().numpy().astype(np.float64)
        vr = max(np.abs(ost.numerics.to_f32(V, "bf16")).max(), np.abs(ost.numerics.to_f32(vob[r], "bf16")).max())
        assert np.all(np.abs(got - O) <= 2.0 ** -8 * 2 * vr + 2.0 ** -8 * np.abs(O) + 1e-6)
        assert np.all(np.abs(lse[r].cpu().numpy() - lse_w) <= 2.0 ** -8)
    st.close()
    del os.environ["HARAG_ATT_SPLIT"]
    # value-distribution guard statistics (R29)
    from oracle import guard
    item = synth.gen_item(2, 2, 64, 64, 5, 1)
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    hr.guard_stats(torch.from_numpy(item.view(np.int16)).cuda(), stats, L=2, H=2, D=64, T=64, gse=(2, 5))
    fl, am = guard.guard_stats(item, "bf16", 2, 5)
    got = stats.cpu().numpy().view(np.uint64)
    assert int(got[0]) == fl and int(got[1]) == int(np.array([am], np.float32).view(np.uint32)[0])
    # analysis kernels
    x = torch.empty(2 * 2 * 64 * 64, dtype=torch.int16, device="cuda")
    synth.gen_item_device(x.data_ptr(), 2, 2, 64, 64, 3, 0)
    hist = hr.exponent_histogram(x, x.numel())
    assert int(hist.sum().item()) == x.numel()
    hr.scheme_error("GSE8", x, L=2, H=2, D=64, T=64)
    torch.cuda.synchronize()
    print(f"sanitize_driver ok ({n} ladders)")


if __name__ == "__main__":
    main()
