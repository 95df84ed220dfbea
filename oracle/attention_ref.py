"""Zamba's shared transformer block ("Zamba ... shared
attention"), plain numpy float64 (TEST INFRASTRUCTURE ONLY).

The block the paper's Zamba experiments run between Mamba layers (Zamba's hybrid layers; the
architecture as in HF transformers modeling_zamba.py ZambaAttentionDecoderLayer + the hybrid
layer's linear, the public definition of the model the paper names):

  x    = RMSNorm_1(concat(h, h0))                 h: the residual stream, h0: the token embeddings
  q, k, v = x W_q^T, x W_k^T, x W_v^T            per head: head_dim = 2 D / H (no rotary embedding)
  o_i  = softmax_j<=i (q_i . k_j / sqrt(head_dim / 2)) v_j      causal, over the KV cache + new keys
  a    = o W_o^T
  y    = RMSNorm_2(a)
  m    = (GELU(y W_g^T) * (y W_u^T)) W_d^T        GELU with erf (exact)
  t    = m W_lin^T                                 the hybrid layer's own linear
The hybrid layer then runs its Mamba layer on RMSNorm(h + t) with residual h.

Tensor parallel (reading Z1): heads are split over the ranks (column-parallel q/k/v,
row-parallel o_proj -> all-reduce), the MLP is split over its intermediate dimension
(column-parallel gate/up, row-parallel down -> all-reduce), the small linear runs replicated.
"""
from __future__ import annotations

import math

import numpy as np


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def rmsnorm(x, w, eps):
    x = _f64(x)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * (1.0 if w is None else _f64(w))


def gelu(x):
    """Exact GELU: x Phi(x) = x (1 + erf(x / sqrt 2)) / 2."""
    x = _f64(x)
    erf = np.vectorize(math.erf)
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def attention(q, K, V, t0, scale):
    """q [B, L, H, d] at positions t0 .. t0+L-1; K, V [B, T, H, d] (T = t0 + L): causal softmax
    attention, o [B, L, H, d]."""
    B, L, H, d = q.shape
    o = np.zeros_like(_f64(q))
    for b in range(B):
        for h in range(H):
            s = (_f64(q[b, :, h]) @ _f64(K[b, :, h]).T) * scale          # [L, T]
            for i in range(L):
                row = s[i, :t0 + i + 1]
                p = np.exp(row - row.max())
                o[b, i, h] = (p / p.sum()) @ _f64(V[b, :t0 + i + 1, h])
    return o


def shared_block(adims, w, h, h0, kv=None, eps=1e-5):
    """adims: d_model, n_heads; w: norm1 [2D], w_q/w_k/w_v [H*d, 2D], w_o [D, H*d], norm2 [D],
    w_g/w_u [I, D], w_d [D, I], w_lin [D, D].  h, h0 [B, L, D].  kv: (K, V) [B, T0, H, d] or None.
    Returns (t [B, L, D], (K', V'))."""
    D, H = adims.d_model, adims.n_heads
    d = 2 * D // H
    h, h0 = _f64(h), _f64(h0)
    B, L, _ = h.shape
    x = rmsnorm(np.concatenate([h, h0], axis=-1), w["norm1"], eps)
    q = (x @ _f64(w["w_q"]).T).reshape(B, L, H, d)
    k = (x @ _f64(w["w_k"]).T).reshape(B, L, H, d)
    v = (x @ _f64(w["w_v"]).T).reshape(B, L, H, d)
    t0 = 0 if kv is None else kv[0].shape[1]
    K = k if kv is None else np.concatenate([_f64(kv[0]), k], axis=1)
    V = v if kv is None else np.concatenate([_f64(kv[1]), v], axis=1)
    o = attention(q, K, V, t0, (d / 2) ** -0.5).reshape(B, L, H * d)
    a = o @ _f64(w["w_o"]).T
    y = rmsnorm(a, w["norm2"], eps)
    m = (gelu(y @ _f64(w["w_g"]).T) * (y @ _f64(w["w_u"]).T)) @ _f64(w["w_d"]).T
    return m @ _f64(w["w_lin"]).T, (K, V)


def shared_block_tp(adims, w, h, h0, k_tp, kv=None, eps=1e-5):
    """The same block on k_tp ranks (reading Z1): rank r owns heads [r H/k, (r+1) H/k) and MLP
    columns [r I/k, (r+1) I/k); the o_proj and down partials are summed in rank order (the two
    all-reduces).  Returns (t, kv shards list)."""
    D, H = adims.d_model, adims.n_heads
    d = 2 * D // H
    I = np.asarray(w["w_g"]).shape[0]
    hk, ik = H // k_tp, I // k_tp
    h, h0 = _f64(h), _f64(h0)
    B, L, _ = h.shape
    x = rmsnorm(np.concatenate([h, h0], axis=-1), w["norm1"], eps)
    a, shards = None, []
    for r in range(k_tp):
        rows = slice(r * hk * d, (r + 1) * hk * d)
        q = (x @ _f64(w["w_q"])[rows].T).reshape(B, L, hk, d)
        k = (x @ _f64(w["w_k"])[rows].T).reshape(B, L, hk, d)
        v = (x @ _f64(w["w_v"])[rows].T).reshape(B, L, hk, d)
        t0 = 0 if kv is None else kv[r][0].shape[1]
        K = k if kv is None else np.concatenate([_f64(kv[r][0]), k], axis=1)
        V = v if kv is None else np.concatenate([_f64(kv[r][1]), v], axis=1)
        o = attention(q, K, V, t0, (d / 2) ** -0.5).reshape(B, L, hk * d)
        p = o @ _f64(w["w_o"])[:, rows].T
        a = p if a is None else a + p                 # all-reduce 1 (rank order)
        shards.append((K, V))
    y = rmsnorm(a, w["norm2"], eps)
    m = None
    for r in range(k_tp):
        cols = slice(r * ik, (r + 1) * ik)
        g = gelu(y @ _f64(w["w_g"])[cols].T) * (y @ _f64(w["w_u"])[cols].T)
        p = g @ _f64(w["w_d"])[:, cols].T
        m = p if m is None else m + p                 # all-reduce 2 (rank order)
    return m @ _f64(w["w_lin"]).T, shards
