"""Oracle of the consumer: attention of a request's query
rows over its assembled KV (TEST INFRASTRUCTURE).

Plain definition in fp64 (R28): for request r, layer l, query head hq (KV head
hq // g) and query row i,

    s_j = scale * <q_i, k_j>          j over the k*T keys, docs in request order
    O_i = sum_j softmax(s)_j v_j,     LSE_i = log sum_j exp(s_j)

where q, k, v are the exact values of the 16-bit inputs (k, v = the oracle's
decoded KV, oracle.store.assemble).  No blocking, no online rescaling.

Prefill form (R30): with the question's own keys / values (n_q tokens, the
TurboRAG prefill's [chunk KV ; question KV]) the keys are the k*T
chunk keys followed by the n_q own keys, and query row i (question token i) sees
every chunk key and own keys 0..i (causal).
"""
from __future__ import annotations

import numpy as np

from . import numerics


def attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float,
              mask: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """q: fp64 [n_q][D]; K, V: fp64 [N][D]; mask: bool [n_q][N] (True = key visible) or None
    -> (O fp64 [n_q][D], LSE fp64 [n_q])."""
    s = scale * (q @ K.T)                                   # [n_q][N]
    if mask is not None:
        s = np.where(mask, s, -np.inf)
    m = s.max(axis=1, keepdims=True)
    e = np.exp(s - m)
    z = e.sum(axis=1, keepdims=True)
    return (e / z) @ V, (m + np.log(z))[:, 0]


def attend_request(Q_bits: np.ndarray, K_bits: np.ndarray, V_bits: np.ndarray, g: int, dtype: str,
                   scale: float | None = None, K_own_bits: np.ndarray | None = None,
                   V_own_bits: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """One request.  Q_bits: uint16 [L][Hl*g][n_q][D]; K_bits, V_bits: uint16 [L][Hl][k*T][D]
    (the assembled KV); K_own_bits, V_own_bits: uint16 [L][Hl][n_q][D] (the question's own keys and
    values: prefill form, causal) or None.  Returns O fp64 [L][Hl*g][n_q][D] and LSE fp64 [L][Hl*g][n_q]."""
    L, HQ, n_q, D = Q_bits.shape
    sc = 1.0 / np.sqrt(D) if scale is None else float(scale)
    q = numerics.to_f32(Q_bits, dtype).astype(np.float64)
    k = numerics.to_f32(K_bits, dtype).astype(np.float64)
    v = numerics.to_f32(V_bits, dtype).astype(np.float64)
    mask = None
    if K_own_bits is not None:
        k = np.concatenate([k, numerics.to_f32(K_own_bits, dtype).astype(np.float64)], axis=2)
        v = np.concatenate([v, numerics.to_f32(V_own_bits, dtype).astype(np.float64)], axis=2)
        n_c = K_bits.shape[2]
        mask = np.ones((n_q, n_c + n_q), dtype=bool)
        mask[:, n_c:] = np.tril(np.ones((n_q, n_q), dtype=bool))
    O = np.empty((L, HQ, n_q, D))
    lse = np.empty((L, HQ, n_q))
    for l in range(L):
        for hq in range(HQ):
            O[l, hq], lse[l, hq] = attention(q[l, hq], k[l, hq // g], v[l, hq // g], sc, mask)
    return O, lse
