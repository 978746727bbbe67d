"""Pins of oracle.codecs.gse_slab_table — step 1 of GSE-8 (§2.2.2:
"exponent distribution range" of a chunk, then the array; R6, R8, R9).

The function reads [Emin, Emax] off a slab's values and hands it to gse_table
(itself pinned by the printed arrays of P:172 / S:147 / S:149 in
test_oracle_codecs.py).  These tests fix the EXTRACTION step against values
whose exponents are known independently of any bit manipulation: every
expectation is a hand-written literal or comes from math.frexp (x = f * 2^e,
0.5 <= f < 1, so the unbiased exponent is e - 1).  A misreading that would
otherwise pass every other test — exponent field 0 counted as -127, fp16
subnormals (fp32-normal numbers) dropped, the sign bit leaking into the
exponent, Emax taken from the largest value instead of the largest magnitude —
fails one of them.
"""
import math

import numpy as np
import pytest

from oracle import codecs, numerics

F32 = np.float32


def unbiased_exponent(v: float) -> int:
    """Exponent E of a nonzero finite v with 2^E <= |v| < 2^(E+1) (library routine, not bits)."""
    return math.frexp(v)[1] - 1


def test_paper_example_values():
    """a chunk whose exponents span [-7, 10] with layout 1+3+4 (step m-1 = 3) gets
    [-7, -4, -1, 2, 5, 8, 10] — here produced from VALUES, not from a given range."""
    x = np.array([2.0 ** -7 * 1.5, 3.0, -2.0 ** 10 * 1.25, 0.0, 40.0, -0.3], dtype=F32)
    assert codecs.gse_slab_table(x, 3, 4) == [-7, -4, -1, 2, 5, 8, 10]


def test_survey_range_default_layout():
    """SURVEY §8(c) hand example: slab exponent range [-13, 4], layout 1+4+3 (step 2) ->
    [-13, -11, -9, -7, -5, -3, -1, 1, 3, 4].  2^-13 and 31.0 (= 1.9375 * 2^4) are the extremes."""
    x = np.array([31.0, -2.0 ** -13, 0.5, -7.0, 2.0 ** -13 * 1.99], dtype=F32)
    assert codecs.gse_slab_table(x, 4, 3) == [-13, -11, -9, -7, -5, -3, -1, 1, 3, 4]


def test_emax_is_largest_magnitude_not_largest_value():
    """A negative value of the largest magnitude sets Emax (the sign is not part of E)."""
    x = np.array([-1000.0, 1.0, 0.25], dtype=F32)            # |-1000| = 1.953 * 2^9
    assert codecs.gse_slab_table(x, 4, 3) == [-2, 0, 2, 4, 6, 8, 9]
    assert unbiased_exponent(-1000.0) == 9 and unbiased_exponent(0.25) == -2


def test_zeros_and_bf16_subnormals_are_ignored():
    """Zeros (both signs) and bf16 subnormals (fp32 exponent field 0) have no exponent to
    share (R9: they encode as 0x00): they must not pull Emin down to -127 or below."""
    bits = np.array([0x0000, 0x8000, 0x0001, 0x807F, 0x0040,      # +0, -0, three bf16 subnormals
                     0x3F80,                                      # 1.0
                     0x4110], dtype=np.uint16)                    # 9.0
    x = numerics.to_f32(bits, "bf16")
    assert [float(v) for v in x[5:]] == [1.0, 9.0]
    assert codecs.gse_slab_table(x, 4, 3) == [0, 2, 3]


def test_smallest_bf16_normal_counts():
    """2^-126 (bf16 0x0080) is normal: it is Emin, and the array (step 2, <= 16 entries)
    is clipped at the top: lo = max(Emin, Emax - 15*2)."""
    bits = np.array([0x0080, 0x3F80, 0x0000], dtype=np.uint16)   # 2^-126, 1.0, 0
    x = numerics.to_f32(bits, "bf16")
    assert unbiased_exponent(float(x[0])) == -126
    assert codecs.gse_slab_table(x, 4, 3) == [-30 + 2 * i for i in range(16)]
    # with a narrow range the clip does not bite and -126 is the first entry
    x2 = np.array([2.0 ** -126, 2.0 ** -120], dtype=F32)
    assert codecs.gse_slab_table(x2, 4, 3) == [-126, -124, -122, -120]


def test_fp16_subnormals_are_fp32_normal():
    """fp16 subnormals (2^-24 .. 2^-15 * 0.999) are exact NORMAL fp32 numbers: their
    exponents are -24..-15 and they take part in [Emin, Emax] (R1: the oracle reads the
    exact fp32 value of the source)."""
    bits = np.array([0x0001, 0x0200, 0x8003, 0x3C00], dtype=np.uint16)   # 2^-24, 2^-15, -3*2^-24, 1.0
    x = numerics.to_f32(bits, "fp16")
    assert [unbiased_exponent(float(v)) for v in x] == [-24, -15, -23, 0]
    assert codecs.gse_slab_table(x, 4, 3) == [-24 + 2 * i for i in range(12)] + [0]
    # ... and the same values round-trip through the encoder at their own exponent
    table = codecs.gse_slab_table(x, 4, 3)
    dec = codecs.gse_decode(codecs.gse_encode(x, table, 4, 3), table, 4, 3)
    assert dec[0] == 2.0 ** -24 and dec[3] == 1.0


def test_single_exponent_and_all_zero():
    """a slab of one exponent gets the one-entry array [E]; an all-zero slab gets none."""
    x = np.array([1.5, -1.25, 1.0, 1.75], dtype=F32)
    assert codecs.gse_slab_table(x, 4, 3) == [0]
    assert codecs.gse_slab_table(np.zeros(8, F32), 4, 3) == []
    assert codecs.gse_slab_table(np.array([0.0, -0.0], F32), 3, 4) == []


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_random_slabs_against_frexp(dtype):
    """Random slabs of 16-bit patterns (zeros and subnormals included): the array equals
    gse_table over [min, max] of frexp exponents of the nonzero values that are normal in
    fp32 (for bf16: |x| >= 2^-126; every nonzero fp16 is fp32-normal)."""
    rng = np.random.default_rng(11)
    top = 0x7F80 if dtype == "bf16" else 0x7C00
    for _ in range(50):
        n = int(rng.integers(1, 300))
        bits = rng.integers(0, top, n).astype(np.uint16) | (rng.integers(0, 2, n) << 15).astype(np.uint16)
        bits[rng.random(n) < 0.2] = 0
        if dtype == "bf16":
            bits[rng.random(n) < 0.1] &= 0x807F                     # subnormals
        x = numerics.to_f32(bits, dtype)
        exps = [unbiased_exponent(float(v)) for v in x if v != 0 and abs(float(v)) >= 2.0 ** -126]
        want = codecs.gse_table(min(exps), max(exps), 4, 3) if exps else []
        assert codecs.gse_slab_table(x, 4, 3) == want
