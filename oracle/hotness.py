"""Oracle hotness: access counting, Algorithm 1 (TEST INFRASTRUCTURE).

Items: item id = 2*doc + kind (kind 0 = K, 1 = V), the paper's 2n chunks
C_1^k, C_1^v, ... (Alg. 1 input).
"""
from __future__ import annotations

import math

import numpy as np


def count_requests(requests, n_docs: int, rank: int = 0, world: int = 1) -> np.ndarray:
    """a1: per-item access counts of a request trace ("obtain access
    frequency statistics"; "counts = number of queries containing
    each id").  Each request touches both items of each of its docs.  Under
    head sharding, request q is counted by rank q mod world only (R20), so the
    SUM over ranks equals the single-rank count."""
    delta = np.zeros(2 * n_docs, dtype=np.int64)
    for q, req in enumerate(requests):
        if q % world != rank:
            continue
        for doc in sorted(set(int(d) for d in req)):
            delta[2 * doc] += 1
            delta[2 * doc + 1] += 1
    return delta


def rank_items(h) -> list[int]:
    """Alg. 1 line 1: sort chunks by access frequency, descending;
    ties by ascending id (R12)."""
    h = [int(v) for v in h]
    return sorted(range(len(h)), key=lambda i: (-h[i], i))


def partition_bounds(M: int, taus) -> list[int]:
    """Alg. 1 lines 2-4: idx_j = tau_j * 2n + idx_{j-1}, floored
    (R11); returns [0, idx_1, ..., idx_{m-1}, M] — the last group takes the
    remainder ("sortedChunks[idx_3 : 2n]")."""
    b = [0]
    for t in taus:
        t = float(t)
        if not (0.0 <= t <= 1.0):
            raise ValueError("tau out of [0,1]")
        b.append(b[-1] + math.floor(t * M))
    if b[-1] > M:
        raise ValueError("taus sum above 1")
    b.append(M)
    return b


def assign_schemes(h, ladder, taus) -> list:
    """Alg. 1: rank, split by thresholds, group j gets ladder[j]
    (S_1 hottest ... S_m coldest).  Returns scheme per item id."""
    if len(taus) != len(ladder) - 1:
        raise ValueError("need len(ladder)-1 thresholds")
    order = rank_items(h)
    b = partition_bounds(len(order), taus)
    scheme = [None] * len(order)
    for j in range(len(ladder)):
        for pos in range(b[j], b[j + 1]):
            scheme[order[pos]] = ladder[j]
    return scheme


def epoch_update(h, delta, decay_shift: int) -> np.ndarray:
    """a9 (R20): h <- (h >> decay_shift) + delta (integer, order-independent)."""
    h = np.asarray(h, dtype=np.int64)
    return (h >> int(decay_shift)) + np.asarray(delta, dtype=np.int64)
