"""Full-size parity (Llama-3-8B KV shape: 32 layers x 8 KV heads x 512 tokens x 128,
16.5 MiB INT8 blobs): every element of whole requests compared with the CPU oracle,
on the host-tier paths that only run at this size and in the launch configuration
bench.py times.

* pageable backing, no pinned tier: every cold item goes pageable -> pinned bounce
  in 4 MiB pieces over the host worker pool -> HBM, the > 4 MiB path;
* disk-backed store (hr_build_from_file, disk_backing): every miss is a multi-piece
  read of the store file into the pinned bounce ("load C_i from Disk"), then a
  re-placement that promotes from disk, immediately followed by requests that stream
  through the same bounce buffers (the promotion-DMA / bounce reuse ordering);
* one whole request of the bench workload (k = 10, 671 MB of KV) and a batch of 32
  requests in one launch of the 2,000-doc HBM-resident bench store (148 persistent
  CTAs, blocked tile ranges): request 0 element by element, one slot (K and V, every
  layer and head) of each of the other 31.

Expected values: tests/oracle_pool.py (the unmodified oracle per item, spread over the
host cores)."""
import numpy as np
import pytest

import synth
from oracle import hotness
from oracle import store as ost
from oracle_pool import expected_items

pytestmark = pytest.mark.gpu

L, H, T, D = 32, 8, 512, 128
NAMES = {"PASS16": ost.PASS16, "INT8": ost.INT8, "FP8E4M3": ost.FP8E4M3, "FP8E5M2": ost.FP8E5M2,
         "GSE8": ost.GSE8, "INT4": ost.INT4}
PAPER = ("INT8", "FP8E4M3", "FP8E5M2", "GSE8")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def gpu_source(alias_R=0):
    def src(doc, kp, vp, stream):
        synth.gen_item_device(kp, L, H, T, D, doc, 0, stream=stream, alias_R=alias_R)
        synth.gen_item_device(vp, L, H, T, D, doc, 1, stream=stream, alias_R=alias_R)
    return src


def job(doc, kind, scheme, alias_R=0):
    return (L, H, T, D, int(doc), kind, int(scheme), "bf16", 0, (4, 3), 0, 1, alias_R)


def check_full(torch, ko, vo, reqs, schemes, slots=None, cache=None, alias_R=0):
    """Compare request r's slots (all of them unless slots[r] is given) element by element."""
    k = reqs.shape[1]
    want = {}
    for r in range(len(reqs)):
        for j in (range(k) if slots is None else slots[r]):
            for kind in (0, 1):
                item = 2 * int(reqs[r, j]) + kind
                if (cache is None or item not in cache) and item not in want:
                    want[item] = job(reqs[r, j], kind, schemes[item], alias_R)
    got_exp = expected_items(want)
    if cache is not None:
        cache.update(got_exp)
        got_exp = cache
    n = 0
    for r in range(len(reqs)):
        gk = ko[r].view(L, H, k * T, D)
        gv = vo[r].view(L, H, k * T, D)
        for j in (range(k) if slots is None else slots[r]):
            for kind, g in ((0, gk), (1, gv)):
                item = 2 * int(reqs[r, j]) + kind
                got = g[:, :, j * T:(j + 1) * T, :].cpu().numpy().view(np.uint16)
                exp = got_exp[item]
                if not np.array_equal(got, exp):
                    bad = np.argwhere(got != exp)
                    raise AssertionError(f"request {r} slot {j} kind {kind} item {item}: {len(bad)} elements "
                                         f"differ, first {bad[:3].tolist()}")
                n += got.size
    return n


def alloc(torch, st, n_req, k):
    nb = st.kv_bytes(k)
    ko = [torch.full((nb // 2,), 0x7FFF, dtype=torch.int16, device="cuda") for _ in range(n_req)]
    vo = [torch.full((nb // 2,), 0x7FFF, dtype=torch.int16, device="cuda") for _ in range(n_req)]
    return ko, vo


def test_fullsize_pageable_bounce_and_disk_tier(torch_cuda, tmp_path):
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    n_docs, k = 8, 3
    lay = ost.Layout(L=L, H=H, T=T, D=D)
    prof = synth.gen_requests(n_docs, 40, k, 1.1, seed=21)
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    taus = (0.25, 0.25, 0.25)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in PAPER], taus)
    sizes = [lay.item_bytes(s) for s in schemes]
    order = hotness.rank_items(h)
    assert min(sizes) > 4 << 20                        # every blob takes the multi-piece paths
    hb = sum(sizes[i] for i in order[:4])              # 4 of 16 items in HBM, the rest streamed
    st = hr.Store(L=L, H=H, D=D, T=T, ladder=PAPER, taus=taus, hbm_budget=hb, pin_budget=0,
                  backing_pinned=False, keep_backing=True, decay_shift=0)
    st.build(n_docs, h, gpu_source())
    assert [st.item_info(i)[0] for i in range(2 * n_docs)] == list(schemes)
    reqs = synth.gen_requests(n_docs, 2, k, 0.3, seed=22)   # flat skew: cold docs are requested
    cache = {}
    ko, vo = alloc(torch, st, 2, k)
    st.assemble(reqs, ko, vo)
    torch.cuda.synchronize()
    s = st.stats()
    assert s["hits"][2] > 0 and s["h2d_items"] > 0      # pageable (PAGE) hits went through the bounce
    check_full(torch, ko, vo, reqs, schemes, cache=cache)

    # the same store on disk: misses are multi-piece reads of the file
    path = str(tmp_path / "full.hr")
    st.save(path)
    st.close()
    ld = hr.Store(L=L, H=H, D=D, T=T, ladder=PAPER, taus=taus, hbm_budget=hb, pin_budget=0,
                  disk_backing=True, keep_backing=False, decay_shift=0)
    ld.build_from_file(path)
    for i in range(2 * n_docs):
        assert ld.item_residency(i) & hr.R_FILE
    ko2, vo2 = alloc(torch, ld, 2, k)
    ld.assemble(reqs, ko2, vo2)
    torch.cuda.synchronize()
    assert ld.stats()["hits_disk"] > 0
    check_full(torch, ko2, vo2, reqs, schemes, cache=cache)

    # an epoch that moves the HBM set onto the cold docs: promotions read the file into the
    # pinned bounce and DMA from it; the very next call streams other cold items through the
    # same bounce buffers — their contents must not be overwritten under the promotion DMA
    by_heat = sorted(range(n_docs), key=lambda d: (-int(h[2 * d] + h[2 * d + 1]), d))
    hot_docs, cold_docs = by_heat[:4], by_heat[4:]
    delta = np.zeros(2 * n_docs, np.int64)
    for d in cold_docs:
        delta[2 * d] = delta[2 * d + 1] = 1000
    ld.hotness_delta().copy_(torch.from_numpy(delta).cuda())
    ld.replace()
    assert ld.stats()["migrations_in"] > 0
    reqs2 = np.array([hot_docs[:k], cold_docs[:k]], dtype=np.uint32)
    ko3, vo3 = alloc(torch, ld, 2, k)
    ld.assemble(reqs2, ko3, vo3)
    torch.cuda.synchronize()
    check_full(torch, ko3, vo3, reqs2, schemes, cache=cache)
    ld.close()


def test_bench_store_full_request_and_batch32(torch_cuda):
    """bench.py's default workload (BASELINE config 1 / SURVEY C2 (i)): 2,000-doc HBM-resident
    store, paper ladder 10/10/10/70 %, batch of 32 requests x k = 10 in ONE assemble launch."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    n_docs, k, B = 2000, 10, 32
    lay = ost.Layout(L=L, H=H, T=T, D=D)
    prof = synth.gen_requests(n_docs, 4 * n_docs, k, 1.1, seed=7, perm_seed=1)   # bench.build_store's profile
    h = hotness.count_requests(prof, n_docs).astype(np.uint64)
    taus = (0.1, 0.1, 0.1)
    schemes = hotness.assign_schemes(h.tolist(), [NAMES[s] for s in PAPER], taus)
    total = sum(lay.item_bytes(s) for s in schemes)
    st = hr.Store(L=L, H=H, D=D, T=T, ladder=PAPER, taus=taus, hbm_budget=total + (1 << 20), keep_backing=False)
    st.build(n_docs, h, gpu_source())
    reqs = synth.gen_requests(n_docs, 8 * B, k, 1.1, seed=1)[:B]          # bench's first batch
    ko, vo = alloc(torch, st, B, k)
    st.assemble(reqs, ko, vo)
    torch.cuda.synchronize()
    assert st.stats()["kernel_launches"] == 1
    cache = {}
    # request 0 whole: 20 items, 335.5 M elements
    n = check_full(torch, ko[:1], vo[:1], reqs[:1], schemes, cache=cache)
    assert n == 2 * L * H * k * T * D
    # one slot of every other request, every layer and head, K and V
    rng = np.random.default_rng(2)
    slots = [[int(rng.integers(k))] for _ in range(B - 1)]
    for c0 in range(0, B - 1, 8):   # bounded host memory for the expected items
        check_full(torch, ko[1 + c0:9 + c0], vo[1 + c0:9 + c0], reqs[1 + c0:9 + c0], schemes,
                   slots=slots[c0:c0 + 8], cache=cache)
        cache.clear()
    st.close()
