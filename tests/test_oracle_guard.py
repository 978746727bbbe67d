"""Pins of oracle/guard.py (the value-distribution guard, R29) against hand-counted slabs,
the closed form R9 states for flushing (E below G_0 - (m-1), zero and subnormals encode 0x00) and the
ladder walk written out by hand.  CPU only."""
import math

import numpy as np
import pytest

from oracle import guard, numerics
from oracle.store import FP8E4M3, FP8E5M2, GSE8, INT4, INT8, PASS16

F32 = np.float32


def bf16(vals):
    return numerics.f32_to_bf16(np.array(vals, dtype=F32))


def test_hand_slab_default_layout():
    """1+4+3 (step 2, 16 entries): Emax = 0 -> lo = -30, values below 2^(lo - 2) = 2^-32 flush.
    2^-31 survives, +-2^-33 flush: 2 (hand count); zeros are not counted."""
    x = np.array([1.0, 2.0 ** -31, 2.0 ** -33, 0.0, -2.0 ** -33, 0.75], dtype=F32)
    assert guard.slab_flushed(x, 4, 3) == 2


def test_hand_slab_short_layout():
    """1+2+5 (step 4, 4 entries): Emax = 1 (3.0) -> lo = 1 - 12 = -11; flush below 2^(-11 - 4) = 2^-15:
    2^-15 survives, 2^-16 and 1.5 * 2^-17 flush."""
    x = np.array([3.0, 2.0 ** -15, 2.0 ** -16, 1.5 * 2.0 ** -17, -1.0], dtype=F32)
    assert guard.slab_flushed(x, 2, 5) == 2
    assert guard.slab_flushed(x, 4, 3) == 0  # the default layout covers 32 binades


def test_subnormals_zeros_and_fp16():
    """bf16 subnormals are fp32 subnormals: always flushed (R9); a slab of zeros flushes nothing; an
    fp16 subnormal is fp32-normal (2^-24) and flushes only if its exponent is out of reach."""
    b = bf16([1.0, 0.5, 0.0])
    b = np.concatenate([b, np.array([0x0001, 0x8002], dtype=np.uint16)])
    assert guard.slab_flushed(numerics.to_f32(b, "bf16"), 4, 3) == 2
    assert guard.slab_flushed(np.zeros(64, F32), 4, 3) == 0
    assert guard.slab_flushed(numerics.to_f32(np.array([0x0001, 0x8003, 0], np.uint16), "bf16"), 4, 3) == 2
    h = np.array([0x3C00, 0x0001], dtype=np.uint16)  # fp16 1.0 and 2^-24
    assert guard.slab_flushed(numerics.to_f32(h, "fp16"), 4, 3) == 0   # -24 >= 0 - 32
    assert guard.slab_flushed(numerics.to_f32(h, "fp16"), 2, 5) == 1   # -24 < 0 - 16


@pytest.mark.parametrize("e_bits,m_bits", [(4, 3), (3, 4), (2, 5)])
def test_closed_form_matches_codec(e_bits, m_bits):
    """The encode/decode count equals R9's closed form: #(nonzero and (fp32 subnormal or
    E < lo - (m - 1))), lo = max(Emin, Emax - (2^e - 1)(m - 1)) over the slab's normals."""
    rng = np.random.default_rng(5 + e_bits)
    for trial in range(40):
        span = int(rng.integers(1, 60))
        ex = rng.integers(-span, 3, size=256)
        x = (rng.uniform(1.0, 2.0, size=256) * np.exp2(ex) * rng.choice([-1, 1], size=256)).astype(F32)
        x[rng.random(256) < 0.05] = 0.0
        b = numerics.f32_to_bf16(x)
        xs = numerics.to_f32(b, "bf16")
        nz = xs[xs != 0]
        E = np.array([math.frexp(float(v))[1] - 1 for v in nz])
        normal = np.abs(nz) >= np.float32(2.0 ** -126)
        if not normal.any():
            want = nz.size
        else:
            step = m_bits - 1
            lo = max(int(E[normal].min()), int(E[normal].max()) - ((1 << e_bits) - 1) * step)
            want = int(np.count_nonzero(~normal | (E < lo - step)))
        assert guard.slab_flushed(xs, e_bits, m_bits) == want, (trial, span)


def test_item_stats_over_all_heads():
    """guard_stats sums the slabs of every (layer, head) and takes max |x| over the item."""
    item = np.zeros((2, 2, 4, 8), dtype=np.uint16)
    item[:] = bf16([1.0])[0]
    item[1, 1, 0, 0] = bf16([2.0 ** -40])[0]     # flushed in its slab (Emax 0, lo -30)
    item[0, 1, 3, 7] = bf16([-448.5])[0]         # bf16 rounds -448.5 to -448.0
    item[1, 0, 2, 2] = bf16([500.0])[0]
    fl, am = guard.guard_stats(item, "bf16", 4, 3)
    assert fl == 1
    assert am == 500.0


def test_ladder_walk():
    lad = [INT8, FP8E4M3, FP8E5M2, GSE8]
    cases = [((GSE8, 3, 1.0), FP8E5M2), ((GSE8, 0, 1.0), GSE8), ((GSE8, 2, 500.0), FP8E5M2),
             ((GSE8, 2, 60000.0), INT8), ((FP8E4M3, 0, 448.0), FP8E4M3), ((FP8E4M3, 0, 448.5), INT8),
             ((FP8E5M2, 0, 57344.0), FP8E5M2), ((FP8E5M2, 0, 57345.0), INT8), ((INT8, 9, 1e30), INT8)]
    for (s, fl, am), want in cases:
        assert guard.guard_schemes([s], [(fl, am)], lad) == [want], (s, fl, am)
    # ladders without the unsafe formats are left alone; a ladder's first scheme is always kept
    assert guard.guard_schemes([INT4, INT8, PASS16], [(5, 1e9)] * 3, [PASS16, INT8, INT4]) == [INT4, INT8, PASS16]
    assert guard.guard_schemes([GSE8], [(7, 1.0)], [GSE8]) == [GSE8]
    assert guard.guard_schemes([GSE8], [(7, 1.0)], [FP8E4M3, GSE8]) == [FP8E4M3]
