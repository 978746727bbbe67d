"""Two ranks, REAL stores (world size 2, KV heads sharded, both processes on cuda:0, gloo for the
collective): each rank assembles its heads of every request and counts only requests q with
q mod 2 == rank (a1); the int64 deltas are SUM-all-reduced (the path's one collective, DESIGN.md
§7) and hr_replace re-ranks and re-places on each rank.  After every epoch both ranks hold the
same placement digest (hr_placement_hash), the same tiers, the tiers the single-process oracle
computes from the summed counts, and outputs equal to the oracle's for their heads."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

L, H, T, D, N_DOCS, K = 2, 4, 64, 64, 24, 4
NORTH = ("PASS16", "INT8", "INT4")


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _budgets(lay, schemes, h):
    from oracle import hotness
    sizes = [lay.item_bytes(s) for s in schemes]
    order = hotness.rank_items(h)
    return sizes, sum(sizes[i] for i in order[:12]), sum(sizes[i] for i in order[12:24])


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2510_20878_b200 as hr
    import synth
    from oracle import hotness
    from oracle import store as ost
    prof = synth.gen_requests(N_DOCS, 80, K, 1.1, seed=7)
    h = hotness.count_requests(prof, N_DOCS).astype(np.uint64)
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype="fp16", rank=rank, world=world)
    names = {"PASS16": ost.PASS16, "INT8": ost.INT8, "INT4": ost.INT4}
    schemes = hotness.assign_schemes(h.tolist(), [names[s] for s in NORTH], (0.25, 0.25))
    sizes, hb, pb = _budgets(lay, schemes, h)
    st = hr.Store(L=L, H=H, D=D, T=T, dtype="fp16", ladder=NORTH, taus=(0.25, 0.25), hbm_budget=hb,
                  pin_budget=pb, rank=rank, world=world, keep_backing=True, decay_shift=1)

    def src(doc, kp, vp, stream):
        synth.gen_item_device(kp, L, H, T, D, doc, 0, dtype="fp16", stream=stream)
        synth.gen_item_device(vp, L, H, T, D, doc, 1, dtype="fp16", stream=stream)

    st.build(N_DOCS, h, src)
    ora = ost.OracleStore(lay, [names[s] for s in NORTH], (0.25, 0.25))
    ora.build(N_DOCS, h, lambda d, kd: synth.gen_item(L, H, T, D, d, kd, heads=lay.heads, dtype="fp16"))
    hashes, tiers, bad = [], [], 0
    nb = st.kv_bytes(K)
    for epoch in range(4):
        reqs = synth.gen_requests(N_DOCS, 30, K, 0.6 + 0.2 * epoch, seed=50 + epoch, perm_seed=60 + epoch)
        ko = [torch.empty(nb // 2, dtype=torch.int16, device="cuda") for _ in reqs]
        vo = [torch.empty(nb // 2, dtype=torch.int16, device="cuda") for _ in reqs]
        st.assemble(reqs, ko, vo)
        torch.cuda.synchronize()
        for r, req in enumerate(reqs):
            Kw, Vw = ora.assemble(list(req))
            bad += not np.array_equal(ko[r].cpu().numpy().view(np.uint16).reshape(Kw.shape), Kw)
            bad += not np.array_equal(vo[r].cpu().numpy().view(np.uint16).reshape(Vw.shape), Vw)
        d = st.hotness_delta().cpu()
        dist.all_reduce(d, op=dist.ReduceOp.SUM)
        st.hotness_delta().copy_(d.cuda())
        st.replace()
        hashes.append(st.placement_hash())
        tiers.append([st.item_info(i)[1] for i in range(2 * N_DOCS)])
    np.save(os.path.join(out_dir, f"tiers{rank}.npy"), np.array(tiers))
    np.save(os.path.join(out_dir, f"hash{rank}.npy"), np.array(hashes, dtype=np.uint64))
    np.save(os.path.join(out_dir, f"bad{rank}.npy"), np.array([bad]))
    st.close()
    dist.destroy_process_group()


def test_two_ranks_real_stores_agree_with_oracle(tmp_path):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    for rank in range(world):
        assert int(np.load(tmp_path / f"bad{rank}.npy")[0]) == 0, f"rank {rank} outputs differ from the oracle"
    t0, t1 = np.load(tmp_path / "tiers0.npy"), np.load(tmp_path / "tiers1.npy")
    assert np.array_equal(t0, t1)
    assert np.array_equal(np.load(tmp_path / "hash0.npy"), np.load(tmp_path / "hash1.npy"))
    # single-process oracle of the epochs (each rank's sizes are equal: same Hl)
    import synth
    from oracle import hotness, placement
    from oracle import store as ost
    prof = synth.gen_requests(N_DOCS, 80, K, 1.1, seed=7)
    h = hotness.count_requests(prof, N_DOCS).astype(np.int64)
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype="fp16", rank=0, world=world)
    names = {"PASS16": ost.PASS16, "INT8": ost.INT8, "INT4": ost.INT4}
    schemes = hotness.assign_schemes(h.tolist(), [names[s] for s in NORTH], (0.25, 0.25))
    sizes, hb, pb = _budgets(lay, schemes, h.astype(np.uint64))
    code = {placement.GPU: 0, placement.PIN: 1, placement.PAGE: 2}
    for epoch in range(4):
        reqs = synth.gen_requests(N_DOCS, 30, K, 0.6 + 0.2 * epoch, seed=50 + epoch, perm_seed=60 + epoch)
        h = hotness.epoch_update(h, hotness.count_requests(reqs, N_DOCS), 1)
        want = [code[t] for t in placement.eager_tiers(h, sizes, hb, pb)]
        assert t0[epoch].tolist() == want, epoch
