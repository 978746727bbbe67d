"""Pins of the oracle codecs against the paper, SPEC.md worked examples,
exhaustive sweeps, closed forms, brute force and library routines.
Citations: P = /root/reference/PAPER.md line, S = SPEC.md line (text copied
into tests/golden/*.txt where a value is printed there)."""
import json
import os
from fractions import Fraction

import ml_dtypes
import numpy as np
import pytest

from oracle import codecs, numerics

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def all_finite_bf16():
    b = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    x = numerics.bf16_to_f32(b)
    ok = np.isfinite(x)
    return b[ok], x[ok]


# ------------------------------------------------------------- bf16 numerics
def test_bf16_examples():
    # S:52
    assert numerics.f32_to_bf16(np.float32([1.0]))[0] == 0x3F80
    assert numerics.bf16_to_f32(np.uint16([0xC000]))[0] == -2.0
    assert numerics.bf16_to_f32(np.uint16([0x0001]))[0] == np.float32(2.0 ** -133)


def test_bf16_roundtrip_all_patterns():
    b, x = all_finite_bf16()
    assert np.array_equal(numerics.f32_to_bf16(x), b)


def test_bf16_rne_overflow_matches_ieee():
    big = np.float32([3.3895314e38, 3.3961e38, 3.4028235e38, -3.4028235e38])
    assert np.array_equal(numerics.f32_to_bf16(big), big.astype(ml_dtypes.bfloat16).view(np.uint16))


def test_bf16_rne_vs_library_and_bruteforce():
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(200000) * rng.choice([1e-3, 1, 30, 1e5], 200000)).astype(np.float32)
    # exact ties
    x[:1000] = numerics.bf16_to_f32(rng.integers(0, 0x7F00, 1000).astype(np.uint16)) * np.float32(1 + 2 ** -8)
    ours = numerics.f32_to_bf16(x)
    lib = x.astype(ml_dtypes.bfloat16).view(np.uint16)
    assert np.array_equal(ours, lib)
    # brute force nearest over all finite bf16 values for a few samples
    _, allx = all_finite_bf16()
    allv = np.unique(allx.astype(np.float64))
    for v in x[:300]:
        d = np.abs(allv - float(v))
        best = allv[d == d.min()]
        got = float(numerics.bf16_to_f32(numerics.f32_to_bf16(np.float32([v])))[0])
        assert got in best


# ---------------------------------------------------------------------- INT8
def test_int8_spec_example():
    # [-2, 1, 0.5, -0.25] -> scale 2/127, payload [-127, 64, 32, -16]
    q, s = codecs.int8_encode(np.float32([[-2.0, 1.0, 0.5, -0.25]]))
    assert s[0] == np.float32(2.0) / np.float32(127.0)
    assert q.tolist() == [[-127, 64, 32, -16]]
    # payload [-127], scale 2/127 -> -2.0 (within one fp32 rounding)
    v = codecs.int8_decode(np.int8([[-127]]), s)
    assert numerics.f32_to_bf16(v)[0, 0] == numerics.f32_to_bf16(np.float32([-2.0]))[0]


def test_int8_zero_group():
    q, s = codecs.int8_encode(np.zeros((1, 8), np.float32))
    assert s[0] == 1.0 and not q.any()


def test_int8_bound_and_bruteforce():
    rng = np.random.default_rng(2)
    x = (rng.standard_normal((400, 16)) * rng.uniform(0.01, 30, (400, 1))).astype(np.float32)
    q, s = codecs.int8_encode(x)
    deq = codecs.int8_decode(q, s).astype(np.float64)
    sf = s.astype(np.float64)[:, None]
    # |x - q*s| <= s/2 (+ one fp32 rounding of the product)
    assert np.all(np.abs(x - deq) <= sf / 2 * (1 + 2 ** -20) + np.abs(deq) * 2 ** -23)
    # q is the argmin over all 255 codes of |x - q s| in exact arithmetic,
    # up to the fp32 rounding of x/s at an exact half (brute force)
    cand = np.arange(-127, 128, dtype=np.float64)
    err = np.abs(x[..., None].astype(np.float64) - cand * sf[..., None])
    best = err.min(-1)
    mine = np.abs(x.astype(np.float64) - q.astype(np.float64) * sf)
    assert np.all(mine <= best + sf * 2 ** -20)
    assert q.min() >= -127  # -128 never produced (R2)


# ---------------------------------------------------------------------- INT4
def test_int4_hand_example():
    x = (np.arange(16, dtype=np.float32) * np.float32(0.5))[None]
    q, s, mn = codecs.int4_encode(x)
    assert s[0] == 0.5 and mn[0] == 0.0
    assert codecs.int4_pack(q).tolist() == [0x10, 0x32, 0x54, 0x76, 0x98, 0xBA, 0xDC, 0xFE]
    assert np.array_equal(codecs.int4_unpack(codecs.int4_pack(q)), q.reshape(-1))
    assert np.array_equal(codecs.int4_decode(q, s, mn), x)


def test_int4_constant_group_and_signed_zero():
    q, s, mn = codecs.int4_encode(np.full((1, 4), -3.5, np.float32))
    assert s[0] == 1.0 and not q.any() and np.all(codecs.int4_decode(q, s, mn) == -3.5)
    q, s, mn = codecs.int4_encode(np.float32([[-0.0, 0.0, 1.0, 2.0]]))
    assert np.signbit(mn[0]) == False  # noqa: E712  (+0 canonical, R4)


def test_int4_range_overflow_saturates():
    """R4: a group spanning (-3e38, 3e38) has an fp32 range that overflows; the
    difference saturates at FLT_MAX (the extremes take codes 0 and 15) and decoding
    stays finite."""
    big = np.float32(3.0e38)
    q, s, mn = codecs.int4_encode(np.float32([[-big, big, 0.0, -big]]))
    assert s[0] == np.float32(np.finfo(np.float32).max) / np.float32(15)
    assert q.tolist() == [[0, 15, 13, 0]]   # 3e38 / (FLT_MAX / 15) = 13.2
    assert np.all(np.isfinite(codecs.int4_decode(q, s, mn)))


def test_int4_bound_and_bruteforce():
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((400, 32)) * rng.uniform(0.01, 30, (400, 1))).astype(np.float32)
    q, s, mn = codecs.int4_encode(x)
    deq = codecs.int4_decode(q, s, mn).astype(np.float64)
    sf, mf = s.astype(np.float64)[:, None], mn.astype(np.float64)[:, None]
    assert np.all(np.abs(x - deq) <= sf / 2 + sf * 2 ** -18 + np.abs(x) * 2 ** -22)
    cand = np.arange(16, dtype=np.float64)
    err = np.abs(x[..., None] - (cand * sf[..., None] + mf[..., None]))
    mine = np.abs(x - (q * sf + mf))
    assert np.all(mine <= err.min(-1) + sf * 2 ** -18)
    assert q.max() <= 15


# ----------------------------------------------------------------------- FP8
def test_fp8_examples():
    g = _gold("fp8_examples.json")
    for variant, cases in g["encode"].items():
        for x, code in cases:
            assert codecs.fp8_encode(np.float32([x]), variant)[0] == int(code, 16), (variant, x)
    assert codecs.fp8_magnitudes("e4m3")[-1] == 448.0
    assert codecs.fp8_magnitudes("e5m2")[-1] == 57344.0    # P:144 "57,334" typo, R5


@pytest.mark.parametrize("variant", ["e4m3", "e5m2"])
def test_fp8_exhaustive_identity(variant):
    # encode(decode(c)) == c for every finite code
    n = codecs.fp8_magnitudes(variant).size
    codes = np.array([c | s for s in (0, 0x80) for c in range(n)], dtype=np.uint8)
    v = codecs.fp8_decode(codes, variant).astype(np.float32)
    assert np.array_equal(codecs.fp8_encode(v, variant), codes)


@pytest.mark.parametrize("variant,lib", [("e4m3", ml_dtypes.float8_e4m3fn), ("e5m2", ml_dtypes.float8_e5m2)])
def test_fp8_vs_library_all_bf16(variant, lib):
    """Nearest-even encoding of every finite bf16 value vs ml_dtypes casts
    (library routine).  Library casts overflow to NaN/inf, so compare in range
    and check saturation separately (R5)."""
    _, x = all_finite_bf16()
    mx = codecs.fp8_magnitudes(variant)[-1]
    ours = codecs.fp8_encode(x, variant)
    inr = np.abs(x) <= mx
    lib_codes = x[inr].astype(lib).view(np.uint8)
    assert np.array_equal(ours[inr], lib_codes)
    assert np.all((ours[~inr] & 0x7F) == codecs.fp8_magnitudes(variant).size - 1)
    assert np.all((ours[~inr] >> 7) == (x[~inr] < 0))


def test_fp8_vs_torch():
    import torch
    rng = np.random.default_rng(4)
    x = (rng.standard_normal(50000) * 40).astype(np.float32)
    x = np.clip(x, -440, 440)
    t = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(codecs.fp8_encode(x, "e4m3"), t)
    t = torch.from_numpy(x).to(torch.float8_e5m2).view(torch.uint8).numpy()
    assert np.array_equal(codecs.fp8_encode(x, "e5m2"), t)


# --------------------------------------------------------------------- GSE-8
def test_gse_paper_array():
    """P:172 prints the array for the worked example: 1+3+4 layout, step 3,
    [-7, -4, -1, 2, 5, 8, 10] (golden/gse_p172.json)."""
    g = _gold("gse_p172.json")
    assert codecs.gse_table(g["emin"], g["emax"], g["e_bits"], g["m_bits"]) == g["array"]


def test_gse_spec_arrays():
    assert codecs.gse_table(0, 9, 3, 4) == [0, 3, 6, 9]
    assert codecs.gse_table(5, 5, 4, 3) == [5]
    t = codecs.gse_table(-40, 10, 3, 4)                       # range too wide: <= 2^e entries
    assert len(t) == 8 and t[-1] == 10 and all(b - a == 3 for a, b in zip(t, t[1:]))


def test_gse_hand_bytes():
    g = _gold("gse_bytes.json")
    for case in g["cases"]:
        t = codecs.gse_table(case["emin"], case["emax"], case["e_bits"], case["m_bits"])
        x = np.float32(case["x"])
        c = codecs.gse_encode(x, t, case["e_bits"], case["m_bits"])
        assert [int(v) for v in c] == [int(v, 16) for v in case["bytes"]], case
        d = codecs.gse_decode(c, t, case["e_bits"], case["m_bits"])
        assert d.tolist() == case["decoded"], case


@pytest.mark.parametrize("e_bits,m_bits", [(4, 3), (3, 4), (2, 5)])
def test_gse_sweep_all_bf16(e_bits, m_bits):
    """S:179 / S:618: every finite bf16 value within the array's coverage keeps
    its sign, never grows in magnitude (truncation), and has relative error
    <= 2^-(m-1-d); zero -> 0."""
    _, x = all_finite_bf16()
    emin, emax = -20, 6
    t = codecs.gse_table(emin, emax, e_bits, m_bits)
    ef = (x.view(np.uint32) >> 23) & 0xFF
    E = ef.astype(np.int64) - 127
    cover = (ef != 0) & (E <= emax) & (E >= t[0] - (m_bits - 1))
    xs = x[cover]
    c = codecs.gse_encode(xs, t, e_bits, m_bits)
    v = codecs.gse_decode(c, t, e_bits, m_bits)
    xd = xs.astype(np.float64)
    assert np.all(np.sign(v) == np.sign(xd))
    assert np.all(np.abs(v) <= np.abs(xd))
    tab = np.array(t)
    G = tab[np.minimum(np.searchsorted(tab, E[cover]), len(t) - 1)]
    d = G - E[cover]
    assert np.all(np.abs(xd - v) / np.abs(xd) <= 2.0 ** -(m_bits - 1 - d))
    # below coverage -> flush to zero
    below = (ef != 0) & (E < t[0] - (m_bits - 1))
    assert not codecs.gse_encode(x[below], t, e_bits, m_bits).any()
    assert codecs.gse_decode(np.uint8([0]), t, e_bits, m_bits)[0] == 0.0


def test_gse_decode_closed_form():
    """Independent pin: with field f != 0 the marker encodes a denormalised
    fraction, so the decoded magnitude is exactly f * 2^(G - (m-1)).  Checked
    for every byte of two layouts against the marker walk of P:163."""
    for e_bits, m_bits in ((4, 3), (3, 4), (2, 5)):
        t = codecs.gse_table(-9, 9, e_bits, m_bits)
        codes = np.arange(256, dtype=np.uint16).astype(np.uint8)
        idx = (codes >> m_bits) & ((1 << e_bits) - 1)
        f = codes & ((1 << m_bits) - 1)
        ok = (idx < len(t)) | (f == 0)
        v = codecs.gse_decode(codes[ok], t, e_bits, m_bits)
        for c, got in zip(codes[ok], v):
            fi = int(c) & ((1 << m_bits) - 1)
            ii = (int(c) >> m_bits) & ((1 << e_bits) - 1)
            want = Fraction(0) if fi == 0 else Fraction(fi) * Fraction(2) ** (t[ii] - (m_bits - 1))
            if c >> 7 and fi:
                want = -want
            assert Fraction(got) == want


def test_gse_corrupt_index():
    t = codecs.gse_table(0, 3, 4, 3)   # 3 entries
    with pytest.raises(ValueError):
        codecs.gse_decode(np.uint8([(10 << 3) | 4]), t, 4, 3)


# ------------------------------------------------------------ RMSE ordering
def test_rmse_examples():
    assert codecs.rmse([1, 2], [1, 2]) == 0.0
    assert abs(codecs.rmse([1, 2], [1, 3]) - np.sqrt(0.5)) < 1e-15


def test_rmse_ordering_on_synthetic_chunks():
    """"INT8 yields the smallest accuracy loss, followed by E4M3 ...
    E5M2 ... GSE-8 results in the highest" — on >= 95% of synthetic chunks."""
    import synth
    good = total = 0
    for doc in range(6):
        for kind in (0, 1):
            bits = synth.gen_item(2, 2, 64, 128, doc, kind)
            for l in range(2):
                for h in range(2):
                    x = numerics.bf16_to_f32(bits[l, h].reshape(-1))
                    q, s = codecs.int8_encode(x.reshape(-1, 128))
                    r8 = codecs.rmse(x, codecs.int8_decode(q, s))
                    r43 = codecs.rmse(x, codecs.fp8_decode(codecs.fp8_encode(x, "e4m3"), "e4m3"))
                    r52 = codecs.rmse(x, codecs.fp8_decode(codecs.fp8_encode(x, "e5m2"), "e5m2"))
                    t = codecs.gse_slab_table(x, 4, 3)
                    rg = codecs.rmse(x, codecs.gse_decode(codecs.gse_encode(x, t, 4, 3), t, 4, 3))
                    good += (r8 <= r43 <= r52 <= rg)
                    total += 1
    assert good >= 0.95 * total
