"""Oracle codecs — PAPER.md §2.2.2 "Low-Precision Data Representation" (TEST INFRASTRUCTURE).

Each encoder takes the exact fp32 values of one group (INT8/INT4) or one
(item, layer, head) slab (FP8, GSE-8) and returns codes + meta; each decoder
returns EXACT values (fp32 for INT8/INT4 — they are defined by fp32 ops —
fp64 for FP8/GSE-8, whose values are exact binary fractions).  Rounding the
decoded value to the output dtype is numerics.round_out.

Readings: R1 group/slab scope, R2 symmetric INT8 ±127,
R3 fp32 IEEE division (no reciprocal, no contraction), R4 INT4 min-max,
R5 FP8 saturation, R6 GSE-8 "rule C" array, R7 step m-1, R9 truncation /
flush, R24 byte bit order.
"""
from __future__ import annotations

import math

import numpy as np

F32 = np.float32

# --------------------------------------------------------------------- INT8
# P:144 "INT8 ... covers a range of [-128, 127]"; symmetric absmax scaling with
# codes in [-127, 127] (R2).


def int8_encode(x: np.ndarray):
    """x: float32 [n_groups][G] -> (q int8 [n_groups][G], s float32 [n_groups]).

    a = max|x| (exact); s = 1 if a == 0 else fl32(a / 127);
    q = clamp(rne(fl32(x / s)), -127, 127).
    """
    x = np.asarray(x, dtype=F32)
    a = np.max(np.abs(x), axis=1)
    s = np.where(a == 0, F32(1.0), a / F32(127.0)).astype(F32)
    q = np.rint(x / s[:, None])
    return np.clip(q, -127, 127).astype(np.int8), s


def int8_decode(q: np.ndarray, s: np.ndarray) -> np.ndarray:
    """fl32(q * s) (one fp32 multiply, R3)."""
    return (np.asarray(q).astype(F32) * np.asarray(s, dtype=F32)[:, None]).astype(F32)


# --------------------------------------------------------------------- INT4
# Not in the paper (P:144 lists 8-bit formats only); north_star asks for
# min-max int4 with bit-packing.  Asymmetric min-max, codes [0, 15] (R4).


def int4_encode(x: np.ndarray):
    """x: float32 [n_groups][G] -> (q uint8 [n_groups][G] in 0..15, s, mn float32).

    mn = min(x) + 0 and mx = max(x) + 0 (the +0 makes a zero extreme +0);
    s = 1 if mx == mn else fl32(sub(mx, mn) / 15);
    q = clamp(rne(fl32(sub(x, mn) / s)), 0, 15),
    where sub(a, b) = min(fl32(a - b), FLT_MAX): a difference of two finite
    values that overflows saturates instead of becoming inf (R4).
    """
    x = np.asarray(x, dtype=F32)
    big = F32(np.finfo(np.float32).max)
    mn = (np.min(x, axis=1) + F32(0.0)).astype(F32)
    mx = (np.max(x, axis=1) + F32(0.0)).astype(F32)
    with np.errstate(over="ignore"):
        d = np.minimum((mx - mn).astype(F32), big)
        s = np.where(mx == mn, F32(1.0), d / F32(15.0)).astype(F32)
        u = np.minimum((x - mn[:, None]).astype(F32), big)
    q = np.rint(u / s[:, None])
    return np.clip(q, 0, 15).astype(np.uint8), s, mn


def int4_decode(q: np.ndarray, s: np.ndarray, mn: np.ndarray) -> np.ndarray:
    """fl32(fl32(q * s) + mn) — two fp32 operations, no fused multiply-add (R4)."""
    qs = (np.asarray(q).astype(F32) * np.asarray(s, dtype=F32)[:, None]).astype(F32)
    return (qs + np.asarray(mn, dtype=F32)[:, None]).astype(F32)


def int4_pack(q: np.ndarray) -> np.ndarray:
    """Element 2i -> low nibble of byte i, element 2i+1 -> high nibble (R24)."""
    q = np.asarray(q, dtype=np.uint8).reshape(-1)
    return (q[0::2] | (q[1::2] << 4)).astype(np.uint8)


def int4_unpack(b: np.ndarray) -> np.ndarray:
    b = np.asarray(b, dtype=np.uint8).reshape(-1)
    out = np.empty(2 * b.size, dtype=np.uint8)
    out[0::2] = b & 0xF
    out[1::2] = b >> 4
    return out


# ---------------------------------------------------------------------- FP8
# P:144 / Fig. fp8-format: E4M3 = 1 sign, 4 exponent, 3 fraction bits, range
# ~[-448, 448]; E5M2 = 1 sign, 5 exponent, 2 fraction bits, range printed as
# "57,334" (a typo: the layout forces 57,344, R5).  E4M3 is the "fn" variant
# (no infinities, S.1111.111 = NaN); E5M2 follows IEEE (exponent 31 = inf/NaN).


def fp8_magnitudes(variant: str) -> np.ndarray:
    """Exact magnitude of every finite non-negative code 0x00..max, ascending (fp64)."""
    if variant == "e4m3":
        ebits, mbits, bias, ncodes = 4, 3, 7, 0x7F      # 0x7F is NaN
    elif variant == "e5m2":
        ebits, mbits, bias, ncodes = 5, 2, 15, 0x7C     # 0x7C.. are inf/NaN
    else:
        raise ValueError(variant)
    mags = []
    for c in range(ncodes):
        e, m = c >> mbits, c & ((1 << mbits) - 1)
        if e == 0:   # subnormal: 0.m * 2^(1-bias)
            mags.append(math.ldexp(m, 1 - bias - mbits))
        else:        # normal: 1.m * 2^(e-bias)
            mags.append(math.ldexp((1 << mbits) + m, e - bias - mbits))
    return np.array(mags, dtype=np.float64)


def fp8_encode(x: np.ndarray, variant: str) -> np.ndarray:
    """Nearest finite code to the exact value, ties to the even code, saturating
    at the largest finite magnitude (448 / 57344); sign bit kept, so negative
    values that round to zero give 0x80 (R5)."""
    mags = fp8_magnitudes(variant)
    x = np.asarray(x, dtype=F32)
    a = np.abs(x.astype(np.float64))
    top = mags.size - 1
    lo = np.clip(np.searchsorted(mags, a, side="right") - 1, 0, top)
    hi = np.minimum(lo + 1, top)
    dlo = a - mags[lo]
    dhi = mags[hi] - a
    take_hi = (hi != lo) & ((dhi < dlo) | ((dhi == dlo) & ((lo & 1) == 1)))
    code = np.where(a >= mags[top], top, np.where(take_hi, hi, lo)).astype(np.uint8)
    sign = np.signbit(x).astype(np.uint8) << 7
    return (code | sign).astype(np.uint8)


def fp8_decode(c: np.ndarray, variant: str) -> np.ndarray:
    """Exact value of each code (fp64)."""
    mags = fp8_magnitudes(variant)
    c = np.asarray(c, dtype=np.uint8)
    m = c & 0x7F
    if np.any(m >= mags.size):
        raise ValueError("non-finite FP8 code")
    v = mags[m]
    return np.where(c & 0x80, -v, v)


# ------------------------------------------------------------------- MXFP8
# SURVEY §8(f) item 4's Blackwell-native cousin of GSE-8's shared exponents (not in the paper; DESIGN.md
# R31): OCP-style microscaling, blocks of 32 consecutive elements share an E8M0 scale 2^(s-127), elements
# are E4M3.  Scale exponent e = floor(log2(max |x|)) - 8 (8 = the exponent of E4M3's largest normal,
# 448 = 1.75 * 2^8), clamped to [-127, 127]; an all-zero block takes e = -127.  Elements: the E4M3 code
# nearest to the exact x * 2^-e (ties to even, saturating at 448: R5); decode = E4M3 value * 2^e.

MX_BLOCK = 32


def mxfp8_encode(x: np.ndarray):
    """x: float32 [n_blocks][32] -> (codes uint8 [n_blocks][32], scales uint8 [n_blocks] = e + 127)."""
    x = np.asarray(x, dtype=F32)
    amax = np.max(np.abs(x.astype(np.float64)), axis=1)
    e = np.full(amax.shape, -127, dtype=np.int64)
    nz = amax > 0
    e[nz] = np.array([math.frexp(float(a))[1] - 1 for a in amax[nz]], dtype=np.int64) - 8  # floor(log2) - 8
    e = np.clip(e, -127, 127)
    y = np.ldexp(x.astype(np.float64), -e[:, None])   # exact in fp64
    codes = fp8_encode(y.astype(F32), "e4m3")         # |y| < 512: fp32 holds it exactly unless |y| < 2^-126
    return codes, (e + 127).astype(np.uint8)


def mxfp8_decode(codes: np.ndarray, scales: np.ndarray) -> np.ndarray:
    """codes uint8 [n_blocks][32], scales uint8 [n_blocks] -> exact values (fp64)."""
    return np.ldexp(fp8_decode(codes, "e4m3"), scales.astype(np.int64)[:, None] - 127)


# -------------------------------------------------------------------- GSE-8
# P:155-172.  A byte is sign | exponent index (e bits) | fraction field (m bits)
# (R24); layouts 1+2+5, 1+3+4, 1+4+3, default 1+4+3.


def gse_table(emin: int, emax: int, e_bits: int, m_bits: int) -> list[int]:
    """Shared-exponent array for exponent range [emin, emax] (R6 "rule C").

    P:172: "divide the distribution range ... into sub-intervals using a fixed
    step size ... use the right endpoint of each interval as the shared
    exponent"; step = m_bits - 1 (the shift may not exceed the fraction bits
    left after the explicit leading 1, R7).  Walk up from lo by the step, last
    entry clipped to emax; lo = max(emin, emax - (2^e - 1)*step) so the array
    has at most 2^e entries (the index must fit in e bits).
    """
    step = m_bits - 1
    lo = max(emin, emax - ((1 << e_bits) - 1) * step)
    n = -(-(emax - lo) // step) + 1
    return [min(lo + i * step, emax) for i in range(n)]


def _f32_fields(x: np.ndarray):
    b = np.asarray(x, dtype=F32).view(np.uint32)
    sign = (b >> np.uint32(31)).astype(np.int64)
    ef = ((b >> np.uint32(23)) & np.uint32(0xFF)).astype(np.int64)
    frac = (b & np.uint32(0x7FFFFF)).astype(np.int64)
    return sign, ef, frac


def gse_slab_table(x: np.ndarray, e_bits: int, m_bits: int) -> list[int]:
    """Array for one slab (P:172 step 1, "exponent distribution range" of the chunk): [Emin, Emax] over the
    nonzero fp32-normal values (R8, R9), then gse_table.  Pinned by tests/test_oracle_gse_slab.py (values
    with known exponents: P:172's example, SURVEY §8(c)'s range, zeros, bf16/fp16 subnormals)."""
    _, ef, _ = _f32_fields(x)
    nz = ef != 0
    if not np.any(nz):
        return []
    e = ef[nz] - 127
    return gse_table(int(e.min()), int(e.max()), e_bits, m_bits)


def gse_encode(x: np.ndarray, table: list[int], e_bits: int, m_bits: int) -> np.ndarray:
    """Encode float32 values with a shared-exponent array.

    Step 1: E = exponent of x.  Step 2: G = smallest shared exponent >= E,
    d = G - E.  Step 3: the m-bit fraction field is the significand 1.f shifted
    right by d (a leading 1 at position d+1 from the MSB, then the top m-1-d
    fraction bits; low bits discarded, i.e. truncation).  Zero and fp32
    subnormals encode as 0x00; E below G_0 - (m-1) flushes to 0x00 (R9).
    """
    x = np.asarray(x, dtype=F32)
    sign, ef, frac = _f32_fields(x)
    out = np.zeros(x.shape, dtype=np.uint8)
    if not table:
        if np.any(ef != 0):
            raise ValueError("empty table for nonzero data")
        return out
    tab = np.array(table, dtype=np.int64)
    E = ef - 127
    idx = np.searchsorted(tab, E, side="left")      # smallest G_i >= E
    if np.any((ef != 0) & (idx >= tab.size)):
        raise ValueError("exponent above the shared-exponent array")
    idxc = np.minimum(idx, tab.size - 1)
    d = tab[idxc] - E
    keep = m_bits - 1 - d                           # fraction bits kept after the marker
    live = (ef != 0) & (keep >= 0)
    keep_s = np.where(live, keep, 0)
    field = (np.int64(1) << keep_s) | (frac >> (23 - keep_s))
    byte = (sign << 7) | (idxc << m_bits) | field
    out[live] = byte[live].astype(np.uint8)
    return out


def gse_decode(c: np.ndarray, table: list[int], e_bits: int, m_bits: int) -> np.ndarray:
    """Decode: the position p of the first 1 in the fraction field gives
    d = p - 1 and E = G[index] - d; the bits after the marker are the fraction
    (left-shifted back).  Field 0 -> +0.  Index past the array -> corrupt."""
    c = np.asarray(c, dtype=np.uint8).astype(np.int64)
    field = c & ((1 << m_bits) - 1)
    idx = (c >> m_bits) & ((1 << e_bits) - 1)
    sign = c >> 7
    nz = field != 0
    if np.any(nz & (idx >= len(table))):
        raise ValueError("corrupt GSE-8 payload: index past the shared-exponent array")
    bitlen = np.array([v.bit_length() for v in range(1 << m_bits)], dtype=np.int64)
    p = m_bits - bitlen[field] + 1                 # 1-indexed marker position from the MSB
    d = p - 1
    tab = np.array(table if table else [0], dtype=np.int64)
    E = tab[np.where(nz, idx, 0)] - d
    nrest = np.maximum(m_bits - p, 0)              # fraction bits after the marker
    rest = field & ((np.int64(1) << nrest) - 1)
    mant = 1.0 + rest.astype(np.float64) / (np.int64(1) << nrest).astype(np.float64)
    v = np.ldexp(mant, E)
    v = np.where(sign == 1, -v, v)
    return np.where(nz, v, 0.0)


def gse_meta(table: list[int], e_bits: int) -> np.ndarray:
    """int8 [2^e]: the array, unused entries -128."""
    m = np.full(1 << e_bits, -128, dtype=np.int8)
    m[: len(table)] = table
    return m


# ------------------------------------------------------------------- metrics
def rmse(x: np.ndarray, xhat: np.ndarray) -> float:
    """Eq. (1): sqrt(1/N sum (x_i - xhat_i)^2), accumulated in fp64."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    y = np.asarray(xhat, dtype=np.float64).reshape(-1)
    if x.shape != y.shape:
        raise ValueError("length mismatch")
    return float(np.sqrt(np.mean((x - y) ** 2)))
