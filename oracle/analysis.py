"""Oracle analysis tooling (TEST INFRASTRUCTURE): exponent distribution of
16-bit KV values (Fig. KV-exponent-range) and the compression error
of Eq. per scheme.

R27: the exponent of a value is its biased exponent field (bf16: 8 bits, bias
127; fp16: 5 bits, bias 15); zeros and subnormals fall in field 0 and
are left out of top-k coverage (they have no exponent to share); top-k
coverage = share of the remaining elements whose field is one of the k most
frequent fields.
"""
from __future__ import annotations

import numpy as np

from . import numerics
from . import store as ost


def exponent_field(bits: np.ndarray, dtype: str) -> np.ndarray:
    """Biased exponent field of 16-bit float bit patterns."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32)
    if dtype == "bf16":
        return (b >> 7) & 0xFF       # 1 sign | 8 exponent | 7 fraction
    if dtype == "fp16":
        return (b >> 10) & 0x1F      # 1 sign | 5 exponent | 10 fraction (IEEE binary16)
    raise ValueError(dtype)


def exponent_histogram(bits: np.ndarray, dtype: str) -> np.ndarray:
    """uint64[256]: count of values per biased exponent field."""
    return np.bincount(exponent_field(bits, dtype).reshape(-1), minlength=256).astype(np.uint64)


def topk_coverage(hist: np.ndarray, k: int) -> float:
    """P:133 "the 8 most frequent exponents can cover ..." (R27: field 0 excluded)."""
    h = np.asarray(hist, dtype=np.float64).copy()
    h[0] = 0.0
    tot = h.sum()
    return float(np.sort(h)[::-1][:k].sum() / tot) if tot else 0.0


def scheme_error(bits: np.ndarray, scheme: int, lay: ost.Layout) -> tuple[float, float]:
    """(sum of squared errors, max |error|) between this rank's heads of one item
    (uint16 [L][H][T][D] of lay.dtype) and its encode -> decode round trip; the
    RMSE of Eq. is sqrt(sse / N) with N = L*Hl*T*D."""
    h0, h1 = lay.heads
    x = np.asarray(bits, dtype=np.uint16).reshape(lay.L, lay.H, lay.T, lay.D)[:, h0:h1]
    blob = ost.encode_item(x, scheme, lay)
    y = ost.decode_item(blob, scheme, lay)
    d = numerics.to_f32(x, lay.dtype).astype(np.float64) - numerics.to_f32(y, lay.dtype).astype(np.float64)
    return float(np.sum(d * d)), float(np.max(np.abs(d))) if d.size else 0.0


def rmse_from(sse: float, n: int) -> float:
    """Eq.: sqrt(1/N sum (x_i - x^_i)^2)."""
    return float(np.sqrt(sse / n))
