"""Test helper: the oracle's expected decoded items at full model shapes, computed in a
pool of host processes (TEST INFRASTRUCTURE).  Each worker runs the unmodified oracle
(synth.gen_item -> oracle.store.encode_item -> decode_item) for one item; the pool only
spreads independent items over the host cores so full-size parity checks (16.5 MiB
blobs, 33.5 MB of decoded KV per item) finish in seconds."""
from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def expected_item(args) -> np.ndarray:
    """uint16 [L][Hl][T][D]: the oracle's decoded item (doc, kind) under `scheme`."""
    (L, H, T, D, doc, kind, scheme, dtype, group, gse, rank, world, alias_R) = args
    import synth
    from oracle import store as ost
    lay = ost.Layout(L=L, H=H, T=T, D=D, dtype=dtype, group=group, gse_e=gse[0], gse_m=gse[1],
                     rank=rank, world=world)
    x = synth.gen_item(L, H, T, D, doc, kind, heads=lay.heads, dtype=dtype, alias_R=alias_R)
    return ost.decode_item(ost.encode_item(x, scheme, lay), scheme, lay)


def expected_items(jobs, procs: int | None = None) -> dict:
    """jobs: {key: args tuple of expected_item}; returns {key: decoded item}."""
    keys = list(jobs)
    procs = procs or min(len(keys), max(1, (os.cpu_count() or 2) - 1))
    if procs <= 1:
        return {k: expected_item(jobs[k]) for k in keys}
    with ProcessPoolExecutor(procs, mp_context=mp.get_context("spawn")) as ex:
        return dict(zip(keys, ex.map(expected_item, [jobs[k] for k in keys])))
