"""Pins of oracle hotness counting, Alg. 1 and Alg. 2 against
SPEC.md's worked examples, hand traces, invariants and an independently
written brute-force interpreter of Alg. 2."""
import itertools
import math
import random

import numpy as np
import pytest

from oracle import hotness, placement
from oracle.placement import DISK, GPU, PAGE, PIN


# ------------------------------------------------------------- a1 counting
def test_count_spec_example():
    # queries [[1,2],[2,3]] -> {1:1, 2:2, 3:1}; items 2*doc+kind
    d = hotness.count_requests([[1, 2], [2, 3]], n_docs=4)
    assert d[2] == 1 and d[4] == 2 and d[6] == 1 and d[3] == 1 and d[5] == 2
    assert d.sum() == 2 * 2 * 2  # S:474 total = queries x k (x2 items per doc)


def test_count_sharded_sum_equals_single():
    rng = np.random.default_rng(0)
    reqs = [rng.choice(50, 5, replace=False) for _ in range(37)]
    full = hotness.count_requests(reqs, 50)
    for world in (2, 3, 8):
        s = sum(hotness.count_requests(reqs, 50, r, world) for r in range(world))
        assert np.array_equal(s, full)


# ------------------------------------------------------------------- Alg. 1
def test_rank_spec_example():
    # {1:5, 2:9, 3:5} -> [2, 1, 3] (id 0 has count 0 -> last)
    assert hotness.rank_items([0, 5, 9, 5]) == [2, 1, 3, 0]
    assert hotness.rank_items([7, 7, 7]) == [0, 1, 2]


@pytest.mark.parametrize("M,taus,sizes", [
    (8, (0.25, 0.25, 0.25), (2, 2, 2, 2)),
    (10, (0.10, 0.10, 0.10), (1, 1, 1, 7)),    # S:316 (P:418 defaults)
    (10, (0.0, 0.0, 0.0), (0, 0, 0, 10)),
    (4381, (0.10, 0.10, 0.10), (438, 438, 438, 3067)),
])
def test_partition_sizes(M, taus, sizes):
    b = hotness.partition_bounds(M, taus)
    assert tuple(b[i + 1] - b[i] for i in range(4)) == sizes


def test_partition_invalid():
    with pytest.raises(ValueError):
        hotness.partition_bounds(10, (0.6, 0.5, 0.0))
    with pytest.raises(ValueError):
        hotness.partition_bounds(10, (-0.1, 0.5, 0.0))


def test_alg1_bruteforce_properties():
    """Brute force on tiny inputs: for every count vector over 5 items with
    counts in 0..3 the assignment is (i) invariant to input order, (ii)
    monotone (hotter never gets a later scheme), (iii) group sizes floor(tau*M)."""
    ladder = ["S1", "S2", "S3", "S4"]
    taus = (0.2, 0.2, 0.4)
    rank_of = {s: i for i, s in enumerate(ladder)}
    for h in itertools.product(range(4), repeat=5):
        a = hotness.assign_schemes(h, ladder, taus)
        for i, j in itertools.permutations(range(5), 2):
            if h[i] > h[j]:
                assert rank_of[a[i]] <= rank_of[a[j]]
        assert [a.count(s) for s in ladder] == [1, 1, 2, 1]
    # order invariance: permuting item ids permutes the assignment (ties by id)
    h = [3, 1, 4, 1, 5, 9, 2, 6]
    sorted_ids = hotness.rank_items(h)
    assert sorted_ids == [5, 7, 4, 2, 0, 6, 1, 3]


def test_epoch_update():
    h = hotness.epoch_update([8, 3, 0], [1, 0, 5], 1)
    assert h.tolist() == [5, 1, 5]


# ------------------------------------------------------------------- Alg. 2
def test_lists_spec_example():
    # 20 ids, (tau_GPU, tau_PIN, tau_PAGE) = (5%, 5%, 10%) -> (1, 1, 2, 16), P:418 defaults
    g, p, a, d = placement.lists_by_fraction(list(range(20)), 0.05, 0.05, 0.10)
    assert (len(g), len(p), len(a), len(d)) == (1, 1, 2, 16)
    g, p, a, d = placement.lists_by_fraction(list(range(20)), 0, 0, 0)
    assert len(d) == 20
    g, p, a, d = placement.lists_by_fraction([3, 1, 0, 2], 0.25, 0.25, 0.25)
    assert (g, p, a, d) == ([3], [1], [0], [2])


def test_lists_by_bytes():
    order = [4, 0, 3, 1, 2]
    sizes = {0: 10, 1: 10, 2: 10, 3: 20, 4: 5}
    g, p, rest = placement.lists_by_bytes(order, sizes, hbm_budget=16, pin_budget=25)
    assert g == [4, 0] and p == [3] and rest == [1, 2]   # 1 would overflow pin: no skipping
    g, p, rest = placement.lists_by_bytes(order, sizes, 0, 0)
    assert g == [] and p == [] and rest == order


def test_lists_by_bytes4():
    """R26: the PAGE_LIST is the next longest prefix that fits the page budget;
    DISK_LIST the rest, order kept."""
    order = [4, 0, 3, 1, 2, 5]
    sizes = {0: 10, 1: 10, 2: 10, 3: 20, 4: 5, 5: 1}
    g, p, a, d = placement.lists_by_bytes4(order, sizes, 16, 25, 15)
    assert (g, p, a, d) == ([4, 0], [3], [1], [2, 5])   # 2 overflows PAGE: 5 (fits) still goes to DISK
    g, p, a, d = placement.lists_by_bytes4(order, sizes, 0, 0, 0)
    assert (g, p, a, d) == ([], [], [], order)
    g, p, a, d = placement.lists_by_bytes4(order, sizes, 0, 0, 10 ** 9)
    assert a == order and d == []
    t = placement.eager_tiers([0, 0, 0, 0, 0, 0], [10] * 6, 10, 10, page_budget=20)
    assert t == ["GPU", "PIN", "PAGE", "PAGE", "DISK", "DISK"]


def _mk(n=4):
    g, p, a, _ = placement.lists_by_fraction(list(range(n)), 0.25, 0.25, 0.25)
    return placement.Alg2(g, p, a, (len(g), len(p), len(a)))


def test_alg2_hand_traces():
    s = _mk()
    assert s.access(0)[0] == DISK          # S:391 rank-0 twice: Disk then GPU
    assert s.access(0)[0] == GPU
    for _ in range(3):
        assert s.access(3)[0] == DISK      # S:392 disk_list never cached
    # S:393 LRU: cap-1 GPU queue holding A; gpu_list item B from disk evicts A
    s = placement.Alg2([10, 11], [], [], (1, 0, 0))
    s.access(10)
    hit, puts, ev = s.access(11)
    assert hit == DISK and puts == [GPU] and ev == [(GPU, 10)]
    # P:246-248 pinned hit of a GPU_LIST item promotes (inclusive: pin copy stays)
    s = placement.Alg2([1], [2], [], (1, 1, 0))
    s.queues[PIN].put(1, 1)
    hit, puts, _ = s.access(1)
    assert hit == PIN and puts == [GPU] and 1 in s.queues[PIN]


def _brute_alg2(gl, pl, al, caps, trace):
    """Independently written interpreter: residency as sets with last-use
    timestamps; LRU victim = argmin timestamp."""
    res = {GPU: {}, PIN: {}, PAGE: {}}
    cap = dict(zip((GPU, PIN, PAGE), caps))
    out = []
    for tick, c in enumerate(trace):
        def put(tier):
            if c in res[tier]:
                res[tier][c] = tick
                return
            if cap[tier] < 1:
                return
            while len(res[tier]) + 1 > cap[tier]:
                victim = min(res[tier], key=lambda k: res[tier][k])
                del res[tier][victim]
            res[tier][c] = tick
        if c in res[GPU]:
            res[GPU][c] = tick
            out.append(GPU)
        elif c in res[PIN]:
            res[PIN][c] = tick
            out.append(PIN)
            if c in gl:
                put(GPU)
        elif c in res[PAGE]:
            res[PAGE][c] = tick
            out.append(PAGE)
            if c in gl:
                put(GPU)
            if c in pl:
                put(PIN)
        else:
            out.append(DISK)
            for tier, lst in ((GPU, gl), (PIN, pl), (PAGE, al)):
                if c in lst:
                    put(tier)
        for t in res:
            assert len(res[t]) <= cap[t]
    return out, {t: set(res[t]) for t in res}


def test_alg2_vs_bruteforce_1000_seeds():
    for seed in range(1000):
        r = random.Random(seed)
        n = r.randint(1, 8)
        order = list(range(n))
        r.shuffle(order)
        fr = [r.choice([0, 0.125, 0.25, 0.5]) for _ in range(3)]
        if sum(fr) > 1:
            fr[2] = 0
        g, p, a, d = placement.lists_by_fraction(order, *fr)
        caps = (len(g), len(p), len(a))
        if r.random() < 0.3:   # smaller caps than lists: LRU really fires
            caps = tuple(max(0, c - r.randint(0, 1)) for c in caps)
        trace = [r.randrange(n) for _ in range(r.randint(1, 32))]
        s = placement.Alg2(g, p, a, caps)
        got = [s.access(c)[0] for c in trace]
        want, res = _brute_alg2(set(g), set(p), set(a), caps, trace)
        assert got == want, seed
        for t in (GPU, PIN, PAGE):
            assert set(s.resident(t)) == res[t]
            assert len(s.resident(t)) <= caps[(GPU, PIN, PAGE).index(t)]
        for c in d:   # S:408 disk-list invisibility
            assert all(c not in s.queues[t] for t in (GPU, PIN, PAGE))


def test_eager_tiers_budget_invariant():
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = int(rng.integers(1, 40))
        h = rng.integers(0, 10, n)
        sizes = rng.choice([100, 200, 50], n)
        hb, pb = int(rng.integers(0, 2000)), int(rng.integers(0, 2000))
        tier = placement.eager_tiers(h, sizes, hb, pb)
        assert sum(int(sizes[i]) for i in range(n) if tier[i] == GPU) <= hb
        assert sum(int(sizes[i]) for i in range(n) if tier[i] == PIN) <= pb
        order = hotness.rank_items(h)
        rank_tier = [tier[i] for i in order]
        seq = [GPU, PIN, PAGE]
        assert [seq.index(t) for t in rank_tier] == sorted(seq.index(t) for t in rank_tier)
