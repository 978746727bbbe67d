"""Pins of the MXFP8 codec (oracle.codecs.mxfp8_*, R31): hand-worked blocks (the scale of a
block whose max is a power of two, saturation past 448 * 2^e, zero blocks, fp32-subnormal maxima at the
-127 clamp), the scale exponent against math.frexp, and the element error bound that follows from
E4M3's spacing.  CPU only."""
import math

import numpy as np

from oracle import codecs
from oracle.store import MXFP8, Layout, decode_slab, encode_slab

F32 = np.float32


def block(vals):
    b = np.zeros((1, 32), dtype=F32)
    b[0, : len(vals)] = vals
    return b


def test_hand_blocks():
    # max 448 = 1.75 * 2^8: e = 0, codes are plain E4M3 (448 -> 0x7E, 1 -> 0x38, -2 -> 0xC0), scale byte 127
    q, s = codecs.mxfp8_encode(block([448.0, 1.0, -2.0]))
    assert s[0] == 127 and list(q[0, :3]) == [0x7E, 0x38, 0xC0]
    assert list(codecs.mxfp8_decode(q, s)[0, :3]) == [448.0, 1.0, -2.0]
    # max 1000: floor(log2 1000) = 9 -> e = 1; 1000 / 2 = 500 saturates to 448 -> decodes to 896; 3 -> 1.5 exact
    q, s = codecs.mxfp8_encode(block([1000.0, 3.0]))
    assert s[0] == 128 and q[0, 0] == 0x7E
    assert list(codecs.mxfp8_decode(q, s)[0, :2]) == [896.0, 3.0]
    # all zeros: e = -127 (scale byte 0), codes 0 (-0 keeps its sign bit)
    q, s = codecs.mxfp8_encode(block([0.0, -0.0]))
    assert s[0] == 0 and q[0, 0] == 0 and q[0, 1] == 0x80 and np.all(q[0, 2:] == 0)
    # max 2^-130 (an fp32 subnormal): floor(log2) - 8 = -138 clamps to -127; x * 2^127 = 2^-3 exactly (0x20)
    q, s = codecs.mxfp8_encode(block([2.0 ** -130]))
    assert s[0] == 0 and q[0, 0] == 0x20 and codecs.mxfp8_decode(q, s)[0, 0] == 2.0 ** -130


def test_scale_exponent_and_error_bound():
    """e + 127 = clamp(frexp(max)[1] - 1 - 8); every element within E4M3's half spacing at its magnitude,
    times 2^e: |x - x^| <= 2^(e-4) * 2^floor(log2|x * 2^-e|) for |x * 2^-e| >= 2^-6, <= 2^(e-10) below."""
    rng = np.random.default_rng(31)
    x = (rng.normal(size=(200, 32)) * np.exp2(rng.integers(-40, 40, size=(200, 1)))).astype(F32)
    q, s = codecs.mxfp8_encode(x)
    amax = np.abs(x.astype(np.float64)).max(axis=1)
    want = np.clip([math.frexp(a)[1] - 1 - 8 for a in amax], -127, 127) + 127
    assert np.array_equal(s.astype(np.int64), want)
    e = s.astype(np.int64)[:, None] - 127
    y = np.abs(x.astype(np.float64)) * np.exp2(-e)
    assert np.all(y < 512)
    err = np.abs(x - codecs.mxfp8_decode(q, s))
    mag = np.floor(np.log2(np.maximum(y, 2.0 ** -6)))
    bound = np.where(y >= 448, np.inf, np.where(y >= 2.0 ** -6, np.exp2(e - 4 + mag), np.exp2(e - 10)))
    assert np.all(err <= bound * (1 + 1e-12))


def test_slab_roundtrip_layout():
    """encode_slab / decode_slab: 1 B per element, one scale byte per 32 elements in the meta record."""
    lay = Layout(L=1, H=1, T=64, D=64, dtype="bf16")
    assert lay.code_bytes(MXFP8) == 4096 and lay.meta_record(MXFP8) == 128
    rng = np.random.default_rng(7)
    from oracle import numerics
    bits = numerics.f32_to_bf16(rng.normal(scale=3.0, size=4096).astype(F32))
    codes, meta = encode_slab(bits, MXFP8, lay)
    assert codes.size == 4096 and meta.size == 128
    out = numerics.to_f32(decode_slab(codes, meta, MXFP8, lay), "bf16")
    x = numerics.to_f32(bits, "bf16")
    assert np.max(np.abs(out - x) / np.maximum(np.abs(x), 2.0 ** -6)) < 2.0 ** -3
