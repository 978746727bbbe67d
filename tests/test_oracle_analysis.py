"""Pins of oracle/analysis.py (exponent histograms P:131-133, RMSE Eq. P:351)."""
import math

import numpy as np

import synth
from oracle import analysis, numerics
from oracle import store as ost


def test_exponent_field_matches_frexp():
    """Brute force: for a normal value v = m * 2^e with m in [0.5, 1) (math.frexp), the
    unbiased exponent is e - 1 and the field is e - 1 + bias; zero / subnormal -> 0."""
    rng = np.random.default_rng(0)
    for dtype, bias, sub_max in (("bf16", 127, 2.0 ** -126), ("fp16", 15, 2.0 ** -14)):
        if dtype == "bf16":
            bits = rng.integers(0, 0x7F80, 4000).astype(np.uint16) | (rng.integers(0, 2, 4000) << 15).astype(np.uint16)
        else:
            bits = rng.integers(0, 0x7C00, 4000).astype(np.uint16) | (rng.integers(0, 2, 4000) << 15).astype(np.uint16)
        vals = numerics.to_f32(bits, dtype).astype(np.float64)
        got = analysis.exponent_field(bits, dtype)
        for v, f in zip(vals, got):
            if v == 0.0 or abs(v) < sub_max:
                assert f == 0
            else:
                assert f == math.frexp(v)[1] - 1 + bias


def test_exponent_hand_values_and_total():
    bits = numerics.f32_to_bf16(np.array([1.0, 0.75, -2.0, 0.0, 24.875], np.float32))
    assert analysis.exponent_field(bits, "bf16").tolist() == [127, 126, 128, 0, 131]
    h = analysis.exponent_histogram(bits, "bf16")
    assert h.sum() == 5 and h[127] == h[126] == h[128] == h[0] == h[131] == 1
    # 16 in field 127 + 2 others: top-1 coverage 16/18, zeros excluded from the denominator
    h = np.zeros(256, np.uint64)
    h[127], h[126], h[128], h[0] = 16, 1, 1, 100
    assert analysis.topk_coverage(h, 1) == 16 / 18 and analysis.topk_coverage(h, 8) == 1.0


def test_synthetic_coverage_like_the_paper():
    """SURVEY §8d measured the generator's top-8 exponent coverage at 98% (K) and 99% (V);
    P:133 reports 96-97% / 95-96% on MS MARCO.  Both well above SPEC's >= 90%."""
    for kind, lo in ((0, 0.97), (1, 0.98)):
        x = synth.gen_item(2, 8, 512, 128, doc=3, kind=kind)
        cov = analysis.topk_coverage(analysis.exponent_histogram(x, "bf16"), 8)
        assert lo <= cov <= 1.0, (kind, cov)


def _one_hot_item(vals, dtype="bf16"):
    lay = ost.Layout(L=1, H=1, T=8, D=32, dtype=dtype, group=32)
    x = np.zeros((1, 1, 8, 32), np.float32)
    x.reshape(-1)[:len(vals)] = vals
    return lay, numerics.round_out(x.reshape(-1), dtype).reshape(x.shape)


def test_scheme_error_hand_int8():
    """INT8, group of 32 holding 1.0 and 0.5 (rest 0): s = fl(1/127) just below 1/127, so
    0.5/s = 63.50000024 -> 64; 64*s = 0.503937... -> bf16 0.50390625 (error 2^-8); 127*s rounds
    to 1.0 in fp32 (error 0).  SSE = 2^-16, max = 2^-8."""
    lay, x = _one_hot_item([1.0, 0.5])
    sse, mx = analysis.scheme_error(x, ost.INT8, lay)
    assert sse == 2.0 ** -16 and mx == 2.0 ** -8


def test_scheme_error_hand_fp8():
    """E4M3: bf16(0.3) = 0.30078125 lies between 0.28125 and 0.3125 (step 2^-5 at exponent -2);
    nearest 0.3125, error 0.01171875.  E5M2 (step 2^-4): candidates 0.25 / 0.3125 -> 0.3125."""
    lay, x = _one_hot_item([0.3])
    for sch in (ost.FP8E4M3, ost.FP8E5M2):
        sse, mx = analysis.scheme_error(x, sch, lay)
        assert mx == 0.01171875 and sse == 0.01171875 ** 2


def test_scheme_error_pass16_zero_and_int8_bound():
    lay = ost.Layout(L=2, H=2, T=16, D=64, group=64)
    x = synth.gen_item(2, 2, 16, 64, doc=1, kind=0)
    assert analysis.scheme_error(x, ost.PASS16, lay) == (0.0, 0.0)
    sse, mx = analysis.scheme_error(x, ost.INT8, lay)
    # |x - deq| <= s/2 + half an output ulp (north_star round-trip bound), s = absmax/127 per group
    a = np.abs(numerics.to_f32(x, "bf16").astype(np.float64)).reshape(-1, 64).max(axis=1)
    assert mx <= (a / 127).max() / 2 + (a.max() * 2.0 ** -9) and sse > 0
    # error ordering of P:349 on this data: INT8 < E4M3 < E5M2 (GSE-8 largest at 1+4+3)
    r = {s: analysis.scheme_error(x, s, lay)[0] for s in (ost.INT8, ost.FP8E4M3, ost.FP8E5M2, ost.GSE8)}
    assert r[ost.INT8] < r[ost.FP8E4M3] < r[ost.FP8E5M2] < r[ost.GSE8]
    assert math.isclose(analysis.rmse_from(sse, x.size), math.sqrt(sse / x.size))
