"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the HA-RAG method: no quantisation, no
ranking, no placement, no counting.  It only produces the inputs both sides
consume, from fixed seeds:

* ``gen_item`` — the bf16/fp16 bit patterns of one KV item (a K or V chunk,
  PAPER.md:185 Alg. 1 input "KVChunks = [C_1^k, C_1^v, ...]"), laid out
  ``[L][H][T][D]``.  Values follow the ranges of PAPER.md:123 (§2.2.1: Keys in
  (-25, 25), Values in (-10, 10)) with an Irwin-Hall bell shape; the recipe is
  DESIGN.md §"Input recipe".  A CUDA copy of the same integer/fp32 recipe lives
  in ``synth/csrc/synth.cu`` (``libharag_synth.so``) so 10k-doc stores can be
  generated on the device; ``tests/test_synth.py`` and the GPU tests cross-check
  the two bit for bit.
* ``gen_requests`` — Zipf(s) retrieval traces of k distinct documents per
  request ("only about 1% of the documents are frequently
  retrieved"), through a seeded permutation of doc ids.

Both generators are pure functions of their seeds.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

CORPUS_SEED = 0x48415241  # "HARA"
KIND_K, KIND_V = 0, 1

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
# fp32 constants of the recipe
K_UNIT = np.float32(4.0 / 37837.0)
V_UNIT = np.float32(2.5 / 37837.0)
K_OUTLIER = np.float32(2.5)
K_CLIP = np.float32(24.875)
V_CLIP = np.float32(9.9375)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def _f32_to_bf16_bits_gen(x: np.ndarray) -> np.ndarray:
    """Generator-private fp32 -> bf16 rounding (nearest-even) for finite x."""
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def gen_item(L: int, H: int, T: int, D: int, doc: int, kind: int, *,
             seed: int = CORPUS_SEED, heads: tuple[int, int] | None = None,
             dtype: str = "bf16", alias_R: int = 0) -> np.ndarray:
    """Bit patterns (uint16) of item (doc, kind), shape [L][h1-h0][T][D].

    gidx is computed over the FULL head count H so a head shard sees exactly
    the values the unsharded store sees.
    """
    h0, h1 = heads if heads is not None else (0, H)
    adoc = doc % alias_R if alias_R else doc
    item = 2 * adoc + kind
    l = np.arange(L, dtype=np.uint64)[:, None, None, None]
    h = np.arange(h0, h1, dtype=np.uint64)[None, :, None, None]
    t = np.arange(T, dtype=np.uint64)[None, None, :, None]
    d = np.arange(D, dtype=np.uint64)[None, None, None, :]
    with np.errstate(over="ignore"):
        gidx = ((((np.uint64(item) * np.uint64(L) + l) * np.uint64(H) + h) * np.uint64(T) + t)
                * np.uint64(D) + d)
        u = splitmix64(np.uint64(seed) ^ gidx)
    m16 = np.uint64(0xFFFF)
    b = ((u & m16) + ((u >> np.uint64(16)) & m16) + ((u >> np.uint64(32)) & m16)
         + (u >> np.uint64(48))).astype(np.int64) - 131070
    bf = b.astype(np.float32)
    if kind == KIND_K:
        x = bf * K_UNIT
        cd = np.where((np.arange(D) % 16) == 0, K_OUTLIER, np.float32(1.0)).astype(np.float32)
        x = (x * cd[None, None, None, :]).astype(np.float32)
        x = np.clip(x, -K_CLIP, K_CLIP)
    else:
        x = bf * V_UNIT
        x = np.clip(x, -V_CLIP, V_CLIP)
    x = x.astype(np.float32)
    if dtype == "bf16":
        return _f32_to_bf16_bits_gen(x)
    if dtype == "fp16":
        return x.astype(np.float16).view(np.uint16)
    raise ValueError(dtype)


QUERY_SEED = 0x51554552  # "QUER"
Q_UNIT = np.float32(1.0 / 37837.0)


def gen_query(n_req: int, L: int, HQ: int, n_q: int, D: int, *, seed: int = QUERY_SEED,
              dtype: str = "bf16") -> np.ndarray:
    """Bit patterns (uint16) of synthetic query rows [n_req][L][HQ][n_q][D] for the attention
    consumer: the same Irwin-Hall counter recipe as gen_item with unit
    standard deviation (scores s = <q, k>/sqrt(D) then have the spread of K's values)."""
    idx = np.arange(n_req * L * HQ * n_q * D, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = splitmix64(np.uint64(seed) ^ idx)
    m16 = np.uint64(0xFFFF)
    b = ((u & m16) + ((u >> np.uint64(16)) & m16) + ((u >> np.uint64(32)) & m16)
         + (u >> np.uint64(48))).astype(np.int64) - 131070
    x = (b.astype(np.float32) * Q_UNIT).astype(np.float32).reshape(n_req, L, HQ, n_q, D)
    if dtype == "bf16":
        return _f32_to_bf16_bits_gen(x)
    if dtype == "fp16":
        return x.astype(np.float16).view(np.uint16)
    raise ValueError(dtype)


def zipf_permutation(n_docs: int, seed: int) -> np.ndarray:
    return np.random.Generator(np.random.PCG64(seed ^ 0x9E3779B9)).permutation(n_docs)


def gen_requests(n_docs: int, n_req: int, k: int, s: float, seed: int,
                 perm_seed: int | None = None) -> np.ndarray:
    """uint32 [n_req][k]: k distinct docs per request, Zipf(s) over doc ranks.

    Rank r (1-based) has probability proportional to r**-s; rank r maps to doc
    perm[r-1] with perm a seeded Fisher-Yates permutation.  Duplicates inside a
    request are redrawn ("k distinct").
    """
    if not (1 <= k <= n_docs):
        raise ValueError("need 1 <= k <= n_docs")
    perm = zipf_permutation(n_docs, seed if perm_seed is None else perm_seed)
    p = np.arange(1, n_docs + 1, dtype=np.float64) ** (-float(s))
    p /= p.sum()
    cdf = np.cumsum(p)
    cdf[-1] = 1.0
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty((n_req, k), dtype=np.uint32)
    for r in range(n_req):
        seen: list[int] = []
        while len(seen) < k:
            draws = np.searchsorted(cdf, rng.random(2 * k), side="right")
            for rk in draws:
                doc = int(perm[min(int(rk), n_docs - 1)])
                if doc not in seen:
                    seen.append(doc)
                    if len(seen) == k:
                        break
        out[r] = seen
    return out


# ---------------------------------------------------------------- CUDA copy
_here = os.path.dirname(os.path.abspath(__file__))
SYNTH_LIB = os.path.join(_here, "libharag_synth.so")
_lib = None


def device_lib():
    """ctypes handle of libharag_synth.so (device copy of gen_item)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SYNTH_LIB):
            raise RuntimeError(f"{SYNTH_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(SYNTH_LIB)
        lib.hrs_gen_item.restype = ctypes.c_int
        lib.hrs_gen_item.argtypes = [
            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32,
            ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def gen_item_device(dst_ptr: int, L: int, H: int, T: int, D: int, doc: int, kind: int, *,
                    seed: int = CORPUS_SEED, heads: tuple[int, int] | None = None,
                    dtype: str = "bf16", alias_R: int = 0, stream: int = 0) -> None:
    """Write gen_item(...) into device memory at dst_ptr ([L][h1-h0][T][D] u16)."""
    h0, h1 = heads if heads is not None else (0, H)
    rc = device_lib().hrs_gen_item(seed, L, H, T, D, h0, h1, doc, kind, alias_R,
                                   1 if dtype == "fp16" else 0, 0,
                                   ctypes.c_void_p(dst_ptr), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"hrs_gen_item failed ({rc})")
