"""CPU tests of the C ABI: the library loads, exports every symbol that
include/harag.h declares, and its host policy (the same C++ the store runs)
equals the oracle on Alg. 1, Alg. 2, counting and epochs."""
import os
import random
import re
import subprocess

import numpy as np
import pytest

import paper_2510_20878_b200 as hr
from oracle import hotness, placement, store as ostore

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "harag.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hr_[a-z0-9_]+)\s*\(", src)) - {"hr_src_fn"})


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", hr._lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hr_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(hr._lib.EXPORTED) <= set(names)
    assert hr.lib.hr_abi_version() == 2


def test_config_validation():
    with pytest.raises(hr.HaragError):
        hr.item_bytes("INT8", L=2, H=2, D=60, T=64)          # D % 8
    with pytest.raises(hr.HaragError):
        hr.item_bytes("INT8", L=2, H=3, D=64, T=64, world=2)  # H % world
    with pytest.raises(hr.HaragError):
        hr.item_bytes("INT8", L=2, H=2, D=64, T=64, group=48)  # power of two
    with pytest.raises(hr.HaragError):
        hr.item_bytes("GSE8", L=2, H=2, D=64, T=64, gse=(5, 2))
    # Alg. 1 needs exactly one tau per ladder boundary; a short list must not leave
    # hr_config_default's thresholds in place or let the C side read past the array
    with pytest.raises(ValueError):
        hr.make_config(L=2, H=2, D=64, T=64, ladder=("INT8", "FP8E4M3", "GSE8"), taus=(0.1,))
    with pytest.raises(ValueError):
        hr.make_config(L=2, H=2, D=64, T=64, ladder=("INT8",) * 7, taus=(0.1,) * 6)
    with pytest.raises(ValueError):
        hr.policy_assign(np.arange(8), ["INT8", "GSE8"], [])
    assert list(hr.policy_assign(np.arange(8), ["INT8", "GSE8"], [0.25])) == [4] * 6 + [1] * 2


@pytest.mark.parametrize("scheme", ["PASS16", "INT8", "FP8E4M3", "FP8E5M2", "GSE8", "INT4", "MXFP8"])
@pytest.mark.parametrize("shape", [(2, 2, 64, 64, 0, 1), (32, 8, 128, 512, 0, 2), (3, 4, 64, 100, 64, 1),
                                   (32, 32, 128, 512, 65536, 1)])
def test_item_bytes_match_oracle_format(scheme, shape):
    L, H, D, T, G, world = shape
    lay = ostore.Layout(L=L, H=H, T=T, D=D, group=G, world=world)
    assert hr.item_bytes(scheme, L=L, H=H, D=D, T=T, group=G, world=world) == \
        lay.item_bytes(ostore.__dict__[scheme])


def test_policy_rank_assign_vs_oracle():
    rng = np.random.default_rng(0)
    ladder = ["INT8", "FP8E4M3", "FP8E5M2", "GSE8"]
    for trial in range(200):
        n = int(rng.integers(1, 300))
        h = rng.integers(0, 6, n).astype(np.uint64)
        taus = list(rng.choice([0.0, 0.05, 0.1, 0.25], 3))
        assert hr.policy_rank(h).tolist() == hotness.rank_items(h)
        got = hr.policy_assign(h, ladder, taus)
        want = hotness.assign_schemes(h.tolist(), [hr.SCHEMES[s] for s in ladder], taus)
        assert got.tolist() == want
    with pytest.raises(hr.HaragError):
        hr.policy_assign(np.zeros(10, np.uint64), ladder, [0.5, 0.5, 0.5])


def test_policy_lists_vs_oracle():
    rng = np.random.default_rng(1)
    for trial in range(200):
        n = int(rng.integers(1, 80))
        h = rng.integers(0, 9, n)
        order = hotness.rank_items(h)
        sizes = rng.choice([16 << 20, 33 << 20, 9 << 20], n).astype(np.uint64)
        hb, pb = int(rng.integers(0, 40)) << 20, int(rng.integers(0, 40)) << 20
        tiers = hr.policy_lists_bytes(order, sizes, hb, pb)
        g, p, rest = placement.lists_by_bytes(order, {i: int(sizes[i]) for i in range(n)}, hb, pb)
        want = np.full(n, 2)
        want[g] = 0
        want[p] = 1
        assert tiers.tolist() == want.tolist()
        gb = int(rng.integers(0, 40)) << 20
        tiers4 = hr.policy_lists_bytes4(order, sizes, hb, pb, gb)
        L4 = placement.lists_by_bytes4(order, {i: int(sizes[i]) for i in range(n)}, hb, pb, gb)
        want = np.empty(n, int)
        for j, lst in enumerate(L4):
            want[lst] = j
        assert tiers4.tolist() == want.tolist()
        f = list(rng.choice([0.0, 0.05, 0.1, 0.2], 3))
        lists = hr.policy_lists_fraction(order, *f)
        L4 = placement.lists_by_fraction(order, *f)
        want = np.empty(n, int)
        for j, lst in enumerate(L4):
            want[lst] = j
        assert lists.tolist() == want.tolist()


def test_policy_count_and_epoch_vs_oracle():
    import synth
    reqs = synth.gen_requests(300, 500, 10, 1.1, seed=3)
    full = hotness.count_requests(reqs, 300)
    assert np.array_equal(hr.policy_count(reqs, 300), full)
    for world in (2, 8):
        s = sum(hr.policy_count(reqs, 300, rank=r, world=world) for r in range(world))
        assert np.array_equal(s, full)
    h = np.arange(600, dtype=np.uint64) * 3
    assert np.array_equal(hr.policy_epoch(h, full, 2), hotness.epoch_update(h.astype(np.int64), full, 2))
    with pytest.raises(hr.HaragError):
        hr.policy_count(np.array([[1, 400]]), 300)


def test_alg2_native_vs_oracle_1000_seeds():
    for seed in range(1000):
        r = random.Random(seed)
        n = r.randint(1, 8)
        order = list(range(n))
        r.shuffle(order)
        fr = [r.choice([0, 0.125, 0.25, 0.5]) for _ in range(3)]
        if sum(fr) > 1:
            fr[2] = 0
        g, p, a, d = placement.lists_by_fraction(order, *fr)
        lst = [3] * n
        for j, L in enumerate((g, p, a)):
            for i in L:
                lst[i] = j
        sizes = [r.choice([1, 2, 3]) for _ in range(n)]
        caps = (r.randint(0, 6), r.randint(0, 6), r.randint(0, 6))
        nat = hr.Alg2(lst, caps, sizes)
        ora = placement.Alg2(g, p, a, caps, sizes)
        names = [placement.GPU, placement.PIN, placement.PAGE, placement.DISK]
        for _ in range(r.randint(1, 32)):
            c = r.randrange(n)
            hit, mask, ev = nat.access(c)
            ohit, oputs, oev = ora.access(c)
            assert names[hit] == ohit, seed
            assert [names[t] for t in range(3) if mask >> t & 1] == sorted(set(oputs), key=names.index)
            assert [(names[t], i) for t, i in ev] == oev
        for t in range(3):
            assert nat.resident(t) == ora.resident(names[t])


def test_policy_guard_vs_oracle():
    """hr_policy_guard (C++) == oracle.guard.guard_schemes on random schemes / statistics, including the
    FP8 saturation boundaries (448, 57344) as exact fp32 bit patterns; a scheme outside the ladder is
    HR_EINVAL."""
    import struct

    from oracle import guard
    rng = np.random.default_rng(29)
    ladders = [["INT8", "FP8E4M3", "FP8E5M2", "GSE8"], ["FP8E5M2", "GSE8"], ["PASS16", "INT8", "INT4"],
               ["GSE8"], ["INT8", "GSE8", "FP8E4M3"]]
    edges = [448.0, np.nextafter(np.float32(448.0), np.float32(1e9)), 57344.0,
             np.nextafter(np.float32(57344.0), np.float32(1e9)), 1.0, 1e6]
    for lad in ladders:
        ids = [hr.SCHEMES[s] for s in lad]
        n = 300
        sc = rng.choice(ids, size=n).astype(np.uint32)
        fl = rng.choice([0, 0, 1, 5], size=n).astype(np.uint64)
        am = np.array([float(rng.choice(edges)) if rng.random() < 0.5 else float(rng.uniform(0, 1e5))
                       for _ in range(n)], dtype=np.float32)
        bits = np.array([struct.unpack("<I", struct.pack("<f", float(a)))[0] for a in am], dtype=np.uint64)
        got = hr.policy_guard(sc, np.stack([fl, bits], axis=1), lad)
        want = guard.guard_schemes([int(x) for x in sc], list(zip(fl.tolist(), am.astype(np.float64).tolist())), ids)
        assert list(got) == want, lad
    with pytest.raises(hr.HaragError):
        hr.policy_guard([hr.SCHEMES["INT4"]], [[0, 0]], ["INT8", "GSE8"])
