"""Oracle numerics: 16-bit float <-> fp32, by definition (TEST INFRASTRUCTURE).

BF16 = 1 sign, 8 exponent (bias 127), 7 fraction bits (§2.2.1 "BF16
format, which consists of 1 sign bit, 8 exponent bits, and 7 fraction bits").
Rounding to BF16/FP16 is round-to-nearest, ties-to-even (R25).
"""
from __future__ import annotations

import numpy as np


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact value of bf16 bit patterns as float32 (bf16 is the top half of fp32)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Nearest bf16 (ties to even) of finite float32 values, as uint16 bits.

    Definition, not a bit trick: the two candidates are the bf16 value obtained
    by truncating x's low 16 bits (``lo``, toward zero) and the next bf16 away
    from zero (``hi``); take the nearer one, and on a tie the one with an even
    last fraction bit.  Distances are exact in fp64.
    """
    x = np.asarray(x, dtype=np.float32)
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite input")
    xb = x.view(np.uint32)
    lo = (xb >> np.uint32(16)).astype(np.uint16)
    hi = (lo.astype(np.uint32) + 1).astype(np.uint16)  # next magnitude, same sign
    xv = x.astype(np.float64)
    dlo = np.abs(xv - bf16_to_f32(lo).astype(np.float64))
    hv = bf16_to_f32(hi).astype(np.float64)
    # IEEE overflow: past the largest finite bf16 the next candidate is inf, which
    # RNE picks from max + ulp/2 on — i.e. treat inf as the value 2^128 here
    hv = np.where(np.isinf(hv), np.copysign(2.0 ** 128, hv), hv)
    dhi = np.abs(xv - hv)
    take_hi = (dhi < dlo) | ((dhi == dlo) & ((lo & 1) == 1))
    return np.where(take_hi, hi, lo).astype(np.uint16)


def fp16_to_f32(bits: np.ndarray) -> np.ndarray:
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float32)


def to_f32(bits: np.ndarray, dtype: str) -> np.ndarray:
    """Exact fp32 value of source-dtype bit patterns (R1)."""
    if dtype == "bf16":
        return bf16_to_f32(bits)
    if dtype == "fp16":
        return fp16_to_f32(bits)
    raise ValueError(dtype)


def round_out(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round exact values (fp32 or fp64 arrays) to the output dtype's bits, RNE.

    fp16 uses numpy's IEEE conversion (round-to-nearest-even, subnormals kept,
    overflow to inf); bf16 uses the definition above.  For fp64 input headed to
    bf16 the value must already be exact in fp32 (true for every decoded value).
    """
    if dtype == "bf16":
        x32 = np.asarray(x).astype(np.float32)
        if np.asarray(x).dtype == np.float64 and not np.array_equal(x32.astype(np.float64), x):
            raise ValueError("value not exact in fp32")
        return f32_to_bf16(x32)
    if dtype == "fp16":
        return np.asarray(x).astype(np.float16).view(np.uint16)
    raise ValueError(dtype)
