"""Multi-process (world size 2, gloo, CPU) tests of the N > 1 host logic: each
rank counts only its own requests (q mod N), the SUM all-reduce of the int64
hotness delta (the path's one collective) gives every rank the
same counts, and the native epoch + re-ranking + byte-budget placement then
agree bit for bit across ranks and with the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2510_20878_b200 as hr
    import synth
    n_docs, k = 300, 10
    h = np.zeros(2 * n_docs, dtype=np.uint64)
    sizes = np.array(hr.policy_assign(np.arange(2 * n_docs), ["INT8", "GSE8"], [0.3]) + 100, dtype=np.uint64)
    base = 0
    placements = []
    for epoch in range(4):
        reqs = synth.gen_requests(n_docs, 64, k, 0.6 + 0.2 * epoch, seed=10 + epoch, perm_seed=20 + epoch)
        delta = hr.policy_count(reqs, n_docs, req_base=base, rank=rank, world=world)
        base += len(reqs)
        t = torch.from_numpy(delta)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        h = hr.policy_epoch(h, t.numpy(), 1)
        order = hr.policy_rank(h)
        tiers = hr.policy_lists_bytes(order, sizes, int(sizes.sum() // 5), int(sizes.sum() // 5))
        placements.append(tiers)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.stack(placements))
    np.save(os.path.join(out_dir, f"h{rank}.npy"), h)
    dist.destroy_process_group()


def test_two_rank_epochs_agree_with_oracle(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    p0, p1 = np.load(tmp_path / "rank0.npy"), np.load(tmp_path / "rank1.npy")
    assert np.array_equal(p0, p1)
    assert np.array_equal(np.load(tmp_path / "h0.npy"), np.load(tmp_path / "h1.npy"))
    # single-process oracle
    import synth
    from oracle import hotness, placement
    import paper_2510_20878_b200 as hr
    n_docs, k = 300, 10
    sizes = np.array(hr.policy_assign(np.arange(2 * n_docs), ["INT8", "GSE8"], [0.3]) + 100, dtype=np.uint64)
    h = np.zeros(2 * n_docs, dtype=np.int64)
    for epoch in range(4):
        reqs = synth.gen_requests(n_docs, 64, k, 0.6 + 0.2 * epoch, seed=10 + epoch, perm_seed=20 + epoch)
        h = hotness.epoch_update(h, hotness.count_requests(reqs, n_docs), 1)
        tiers = placement.eager_tiers(h, [int(x) for x in sizes], int(sizes.sum() // 5), int(sizes.sum() // 5))
        want = [{placement.GPU: 0, placement.PIN: 1, placement.PAGE: 2}[t] for t in tiers]
        assert p0[epoch].tolist() == want, epoch
