"""The shared synthetic generator: ranges of P:123, determinism, Zipf trace."""
import numpy as np

import synth
from oracle import numerics


def test_item_ranges_and_determinism():
    k = synth.gen_item(2, 4, 128, 128, 5, synth.KIND_K)
    v = synth.gen_item(2, 4, 128, 128, 5, synth.KIND_V)
    assert np.array_equal(k, synth.gen_item(2, 4, 128, 128, 5, synth.KIND_K))
    kf, vf = numerics.bf16_to_f32(k), numerics.bf16_to_f32(v)
    assert np.abs(kf).max() <= 24.875 and np.abs(vf).max() <= 9.9375
    # exponent concentration (top-8 exponents cover 95-97%; S:562 >= 0.90)
    for x in (kf, vf):
        e = ((x.view(np.uint32) >> 23) & 0xFF)[x != 0]
        cnt = np.sort(np.bincount(e))[::-1]
        assert cnt[:8].sum() / cnt.sum() >= 0.90
    assert not np.array_equal(k, synth.gen_item(2, 4, 128, 128, 6, synth.KIND_K))


def test_alias_and_heads():
    a = synth.gen_item(1, 4, 8, 16, 13, 1, alias_R=5)
    assert np.array_equal(a, synth.gen_item(1, 4, 8, 16, 3, 1))
    assert np.array_equal(synth.gen_item(1, 4, 8, 16, 2, 0, heads=(1, 3)),
                          synth.gen_item(1, 4, 8, 16, 2, 0)[:, 1:3])


def test_requests_distinct_and_skewed():
    r = synth.gen_requests(2000, 4096, 10, 1.1, seed=1)
    assert r.shape == (4096, 10)
    assert all(len(set(row)) == 10 for row in r)
    assert np.array_equal(r, synth.gen_requests(2000, 4096, 10, 1.1, seed=1))
    c = np.bincount(r.reshape(-1), minlength=2000)
    top = np.sort(c)[::-1][:20].sum() / c.sum()
    assert top >= 0.30                                   # top 1% >= 30%
