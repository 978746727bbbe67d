"""Pins of oracle/attention.py against closed forms, invariants and an
independent library implementation (torch's scaled_dot_product_attention in
fp64 on the CPU)."""
import math

import numpy as np
import pytest

from oracle import attention, numerics


def test_uniform_scores_give_the_mean_and_log_n():
    """Equal keys -> equal weights: O = mean of V, LSE = s + log N."""
    rng = np.random.default_rng(0)
    q = rng.normal(size=(3, 16))
    k = np.tile(rng.normal(size=(1, 16)), (10, 1))
    v = rng.normal(size=(10, 16))
    O, lse = attention.attention(q, k, v, 0.25)
    assert np.allclose(O, v.mean(axis=0)[None, :], atol=1e-14)
    assert np.allclose(lse, 0.25 * (q @ k[0]) + math.log(10), atol=1e-13)


def test_dominant_key_selects_its_value():
    q = np.zeros((1, 4))
    q[0, 0] = 1.0
    k = np.zeros((5, 4))
    k[3, 0] = 100.0
    v = np.arange(20.0).reshape(5, 4)
    O, lse = attention.attention(q, k, v, 1.0)
    assert np.allclose(O[0], v[3], atol=1e-30) and abs(lse[0] - 100.0) < 1e-12


def test_two_keys_closed_form():
    """softmax of (a, b) = (1/(1+e^(b-a)), ...): O = w v0 + (1-w) v1, LSE = log(e^a + e^b)."""
    q = np.array([[1.0, 2.0]])
    k = np.array([[0.5, 0.0], [0.0, 1.0]])
    v = np.array([[1.0, 0.0], [0.0, 1.0]])
    a, b = 0.5, 2.0
    w = 1.0 / (1.0 + math.exp(b - a))
    O, lse = attention.attention(q, k, v, 1.0)
    assert np.allclose(O[0], [w, 1 - w], atol=1e-15) and abs(lse[0] - math.log(math.exp(a) + math.exp(b))) < 1e-14


def test_matches_torch_sdpa_fp64_with_gqa():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    L, H, g, n_q, N, D = 2, 2, 4, 5, 96, 64
    Qb = numerics.f32_to_bf16(rng.normal(size=(L, H * g, n_q, D)).astype(np.float32))
    Kb = numerics.f32_to_bf16((4 * rng.normal(size=(L, H, N, D))).astype(np.float32))
    Vb = numerics.f32_to_bf16(rng.normal(size=(L, H, N, D)).astype(np.float32))
    O, lse = attention.attend_request(Qb, Kb, Vb, g, "bf16")
    q = torch.from_numpy(numerics.to_f32(Qb, "bf16").astype(np.float64))
    k = torch.from_numpy(numerics.to_f32(Kb, "bf16").astype(np.float64)).repeat_interleave(g, dim=1)
    v = torch.from_numpy(numerics.to_f32(Vb, "bf16").astype(np.float64)).repeat_interleave(g, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v).numpy()
    assert np.allclose(O, ref, rtol=0, atol=1e-12)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(D)
    assert np.allclose(lse, torch.logsumexp(s, dim=-1).numpy(), atol=1e-12)


def test_weights_are_a_convex_combination():
    """Every output lies inside the per-column range of V (softmax weights >= 0, sum 1)."""
    rng = np.random.default_rng(5)
    q, k, v = rng.normal(size=(7, 32)), 3 * rng.normal(size=(50, 32)), rng.normal(size=(50, 32))
    O, _ = attention.attention(q, k, v, 1 / math.sqrt(32))
    assert np.all(O <= v.max(axis=0) + 1e-12) and np.all(O >= v.min(axis=0) - 1e-12)


def test_prefill_own_block_matches_torch_sdpa_masked():
    """Prefill form (R30): [chunk keys ; own keys] with the causal mask on the own block — against torch
    SDPA in fp64 with the same boolean mask written out (a library routine, the special case of masked
    attention), and row 0 against the explicit formula over the chunk keys plus own key 0 only."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(30)
    L, H, g, n_q, N, D = 2, 2, 3, 6, 64, 32
    Qb = numerics.f32_to_bf16(rng.normal(size=(L, H * g, n_q, D)).astype(np.float32))
    Kb = numerics.f32_to_bf16((3 * rng.normal(size=(L, H, N, D))).astype(np.float32))
    Vb = numerics.f32_to_bf16(rng.normal(size=(L, H, N, D)).astype(np.float32))
    Ko = numerics.f32_to_bf16((3 * rng.normal(size=(L, H, n_q, D))).astype(np.float32))
    Vo = numerics.f32_to_bf16(rng.normal(size=(L, H, n_q, D)).astype(np.float32))
    O, lse = attention.attend_request(Qb, Kb, Vb, g, "bf16", K_own_bits=Ko, V_own_bits=Vo)
    f = lambda b: torch.from_numpy(numerics.to_f32(b, "bf16").astype(np.float64))  # noqa: E731
    q = f(Qb)
    k = torch.cat([f(Kb), f(Ko)], dim=2).repeat_interleave(g, dim=1)
    v = torch.cat([f(Vb), f(Vo)], dim=2).repeat_interleave(g, dim=1)
    m = torch.ones(n_q, N + n_q, dtype=torch.bool)
    for i in range(n_q):
        m[i, N + i + 1:] = False
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=m).numpy()
    assert np.allclose(O, ref, rtol=0, atol=1e-12)
    # row 0, layer 0, query head 0: softmax over the N chunk scores and own key 0, written out
    qq, kk, vv = q[0, 0, 0].numpy(), k[0, 0, :N + 1].numpy(), v[0, 0, :N + 1].numpy()
    s = kk @ qq / math.sqrt(D)
    w = np.exp(s - s.max())
    assert np.allclose(O[0, 0, 0], (w / w.sum()) @ vv, atol=1e-12)
    assert abs(lse[0, 0, 0] - (s.max() + math.log(w.sum()))) < 1e-12
