"""GPU analysis tooling against the oracle: exponent
histograms bit-exact (integer counts), scheme error (Eq. P:351) with the max
|error| exact and the fp64 sum of squares within summation-order rounding."""
import numpy as np
import pytest

import synth
from oracle import analysis
from oracle import store as ost

pytestmark = pytest.mark.gpu

SCH = {"PASS16": ost.PASS16, "INT8": ost.INT8, "FP8E4M3": ost.FP8E4M3, "FP8E5M2": ost.FP8E5M2,
       "GSE8": ost.GSE8, "INT4": ost.INT4}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _dev(torch, bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda()


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("n,offset", [(2 * 4 * 64 * 128, 0), (12345, 0), (777, 3), (0, 0), (8, 1)])
def test_exponent_histogram_exact(torch_cuda, dtype, n, offset):
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    x = synth.gen_item(2, 4, 64, 128, doc=5, kind=0, dtype=dtype).reshape(-1)
    x = np.concatenate([x, np.array([0, 0x8000, 0x7F7F, 0x0001], np.uint16)])[:n + offset + 4]
    t = _dev(torch, x)
    h = hr.exponent_histogram(t[offset:offset + n] if n else t[:0], n, dtype=dtype)
    torch.cuda.synchronize()
    want = analysis.exponent_histogram(x[offset:offset + n], dtype) if n else np.zeros(256, np.uint64)
    assert np.array_equal(h.cpu().numpy().astype(np.uint64), want)


def test_exponent_histogram_accumulates_and_full_item(torch_cuda):
    """One Llama-3-8B-shaped item (16.8M values), then a second call accumulating into it."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    x = synth.gen_item(32, 8, 512, 128, doc=11, kind=1)
    t = _dev(torch, x)
    h = hr.exponent_histogram(t, x.size)
    hr.exponent_histogram(t, x.size, hist=h)
    torch.cuda.synchronize()
    assert np.array_equal(h.cpu().numpy().astype(np.uint64), 2 * analysis.exponent_histogram(x, "bf16"))


@pytest.mark.parametrize("scheme", list(SCH))
@pytest.mark.parametrize("geo", [dict(L=2, H=2, T=64, D=128, dtype="bf16"),
                                 dict(L=3, H=4, T=32, D=64, dtype="fp16", group=32, rank=1, world=2),
                                 dict(L=2, H=2, T=64, D=64, dtype="bf16", gse=(3, 4))])
def test_scheme_error_matches_oracle(torch_cuda, scheme, geo):
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    g = dict(geo)
    gse = g.pop("gse", (4, 3))
    lay = ost.Layout(L=g["L"], H=g["H"], T=g["T"], D=g["D"], dtype=g["dtype"], group=g.get("group", 0),
                     gse_e=gse[0], gse_m=gse[1], rank=g.get("rank", 0), world=g.get("world", 1))
    for kind in (0, 1):
        x = synth.gen_item(g["L"], g["H"], g["T"], g["D"], doc=7, kind=kind, dtype=g["dtype"])
        sse, mx = hr.scheme_error(scheme, _dev(torch, x), gse=gse, **g)
        want_sse, want_mx = analysis.scheme_error(x, SCH[scheme], lay)
        assert mx == want_mx
        assert sse == pytest.approx(want_sse, rel=1e-12, abs=0.0)


def test_scheme_error_full_shape_and_nan(torch_cuda):
    """Full Llama-3-8B item for INT8 and E4M3 (oracle finishes in seconds); NaN rejected."""
    import paper_2510_20878_b200 as hr
    torch = torch_cuda
    x = synth.gen_item(32, 8, 512, 128, doc=2, kind=0)
    lay = ost.Layout(L=32, H=8, T=512, D=128)
    t = _dev(torch, x)
    for s in ("INT8", "FP8E4M3"):
        sse, mx = hr.scheme_error(s, t, L=32, H=8, T=512, D=128)
        want = analysis.scheme_error(x, SCH[s], lay)
        assert mx == want[1] and sse == pytest.approx(want[0], rel=1e-12)
    y = x.copy()
    y[5, 3, 100, 7] = 0x7FC0
    with pytest.raises(hr.HaragError, match="EINVAL"):
        hr.scheme_error("INT8", _dev(torch, y), L=32, H=8, T=512, D=128)
