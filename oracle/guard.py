"""Oracle of the value-distribution guard (TEST INFRASTRUCTURE; only tests/, smoke() and bench.py's
cpu_baseline may import it).

SURVEY §8(f) item 4 (an extra the paper does not have; R29): Alg. 1 picks a
chunk's scheme from its hotness alone, but two of the paper's formats can lose a chunk's values
outright:
  * GSE-8: a value whose exponent lies more than m-1 below the first shared exponent of
    its slab's array encodes as field 0 (R9: truncation; zero and subnormals encode 0x00), i.e. it is
    FLUSHED to zero.  The array covers at most (2^e - 1)(m - 1) + (m - 1) binades below Emax (rule C,
    R6), so a slab whose exponent range is wider flushes its smallest values;
  * FP8: E4M3 saturates above 448, E5M2 above 57344 (R5).
The guard measures both per item and moves an item whose scheme would lose values one step towards
the hot end of the ladder (the more precise formats), repeatedly, never past the ladder's first
scheme.  Everything here follows the definitions with the oracle's own codecs; no shortcut of the
GPU path (a closed-form flush threshold) is used.
"""
from __future__ import annotations

import numpy as np

from . import codecs, numerics
from .store import FP8E4M3, FP8E5M2, GSE8

FP8_MAX = {FP8E4M3: 448.0, FP8E5M2: 57344.0}  # largest finite magnitudes (R5; P:144 prints 448, "57,334")


def slab_flushed(x: np.ndarray, e_bits: int, m_bits: int) -> int:
    """Nonzero values of one slab (float32) whose GSE-8 code decodes to 0: encode with the slab's own
    shared-exponent array (gse_slab_table) and decode, both from oracle.codecs."""
    x = np.asarray(x, dtype=np.float32).ravel()
    table = codecs.gse_slab_table(x, e_bits, m_bits)
    if not table:  # no normal value at all: every nonzero value (a subnormal) encodes 0x00 (R9)
        return int(np.count_nonzero(x))
    dec = codecs.gse_decode(codecs.gse_encode(x, table, e_bits, m_bits), table, e_bits, m_bits)
    return int(np.count_nonzero((x != 0) & (dec == 0)))


def guard_stats(bits: np.ndarray, dtype: str, e_bits: int, m_bits: int) -> tuple[int, float]:
    """(flushed, absmax) of one item: bits = its 16-bit source values [L][H][T][D] over ALL heads (the
    statistic must not depend on how heads are sharded, so every rank derives the same schemes).
    flushed = sum over the (layer, head) slabs of slab_flushed; absmax = max |x| (fp32)."""
    x = numerics.to_f32(np.asarray(bits), dtype)
    L, H = x.shape[0], x.shape[1]
    flushed = sum(slab_flushed(x[l, h], e_bits, m_bits) for l in range(L) for h in range(H))
    return flushed, float(np.max(np.abs(x))) if x.size else 0.0


def unsafe(scheme: int, flushed: int, absmax: float) -> bool:
    """Would `scheme` lose values of an item with these statistics?"""
    if scheme == GSE8:
        return flushed > 0
    if scheme in FP8_MAX:
        return absmax > FP8_MAX[scheme]
    return False  # PASS16, INT8, INT4 represent every finite value's magnitude range


def guard_schemes(schemes, stats, ladder) -> list[int]:
    """Alg. 1's schemes -> guarded schemes: while an item's scheme is unsafe for it and is not the
    ladder's first, take the previous (hotter) ladder scheme."""
    ladder = list(ladder)
    out = []
    for s, (fl, am) in zip(schemes, stats):
        p = ladder.index(s)
        while p > 0 and unsafe(ladder[p], fl, am):
            p -= 1
        out.append(ladder[p])
    return out
