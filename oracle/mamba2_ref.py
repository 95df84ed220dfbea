"""Mamba-2 (SSD) mixer, plain numpy float64 (TEST INFRASTRUCTURE ONLY).

PAPER.md:116 (Mamba-2 "reformulates the Mamba mixer's state-update computation"), 367 ("Mamba-2
preserves the same high-level mixer pipeline (projection, convolution, state update, gating,
output projection), so we reuse the same sharding and communication principles and only adapt to
the specific packed parameter layout").  The mixer, as in the public model definition (HF
transformers modeling_mamba2.py; the SSD paper's scalar-A-per-head selective SSM), written here as
the literal per-timestep recurrence:

  [z | x | B | C | dt] = x_in W_in^T                  E = d_inner, G groups of N states, H heads of P
  [x | B | C] <- SiLU(causal depthwise conv1d over the x, B, C channels)
  dt_h = softplus(dt_h + dt_bias_h);  A_h = -exp(A_log_h)
  for t: h[h, p, n] <- exp(dt_h A_h) h[h, p, n] + dt_h x[h, p] B[g(h), n]
         y[h, p] = sum_n C[g(h), n] h[h, p, n] + D_h x[h, p]
  g = y * SiLU(z);  o = g / sqrt(mean(g^2) + eps) * w_norm   (gated RMSNorm over d_inner, norm
                                                                after the gate, as HF's
                                                                MambaRMSNormGated)
  out = residual + o W_out^T
State carried prefill -> decode: (conv window of the x|B|C channels, h [B, H, P, N]).

Tensor parallel (reading M1): heads split over the ranks (z, x, dt rows and the conv /
dt_bias / A_log / D / norm-weight entries of the owned heads; W_out columns), B and C replicated
when n_groups does not split (they come straight from the packed in_proj, so no all-reduce is
needed before the scan -- one collective fewer than Mamba-1's x_proj), the gated RMSNorm's sum of
squares all-reduced over the ranks (M floats), out_proj row-parallel -> all-reduce.
"""
from __future__ import annotations

import numpy as np


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def silu(x):
    x = _f64(x)
    return x / (1.0 + np.exp(-x))


def softplus(x):
    x = _f64(x)
    return np.where(x > 20.0, x, np.log1p(np.exp(np.minimum(x, 20.0))))


def zero_state(batch, d, heads, headdim, d_state, d_conv, conv_dim):
    return np.zeros((batch, conv_dim, d_conv - 1)), np.zeros((batch, heads, headdim, d_state))


def mixer_forward(m2, w, x_in, residual, state=None):
    """m2: d_model, d_inner, d_state, headdim, n_groups, d_conv, eps.  w: w_in [2E + 2GN + H, D],
    conv_w [E + 2GN, K], conv_b [E + 2GN], dt_bias [H], a_log [H], d_skip [H], norm_w [E],
    w_out [D, E].  x_in, residual [B, L, D].  Returns (out, (conv_state, h))."""
    x_in, residual = _f64(x_in), _f64(residual)
    Bsz, L, D = x_in.shape
    E, N, P, G, K = m2.d_inner, m2.d_state, m2.headdim, m2.n_groups, m2.d_conv
    H = E // P
    conv_dim = E + 2 * G * N
    if state is None:
        state = zero_state(Bsz, D, H, P, N, K, conv_dim)
    conv_state, h = _f64(state[0]), _f64(state[1]).copy()
    proj = x_in @ _f64(w["w_in"]).T
    z = proj[..., :E]
    xbc = proj[..., E:E + conv_dim]
    dt = proj[..., E + conv_dim:]
    # causal depthwise conv (cross-correlation, tap K-1 = current token) over the cached window
    xt = np.concatenate([np.transpose(conv_state, (0, 2, 1)), xbc], axis=1)     # [B, K-1+L, C]
    cw = _f64(w["conv_w"])
    xc = np.zeros_like(xbc)
    for j in range(K):
        xc += xt[:, j:j + L, :] * cw[:, j]
    xc += _f64(w["conv_b"])
    u = silu(xc)
    conv_new = np.transpose(xt[:, L:L + K - 1, :], (0, 2, 1)).copy()
    x = u[..., :E].reshape(Bsz, L, H, P)
    Bm = u[..., E:E + G * N].reshape(Bsz, L, G, N)
    Cm = u[..., E + G * N:].reshape(Bsz, L, G, N)
    dt = softplus(dt + _f64(w["dt_bias"]))                                        # [B, L, H]
    A = -np.exp(_f64(w["a_log"]))                                                  # [H]
    Dsk = _f64(w["d_skip"])
    grp = np.arange(H) // (H // G)
    y = np.zeros((Bsz, L, H, P))
    for t in range(L):
        dA = np.exp(dt[:, t] * A)                                                  # [B, H]
        Bt = Bm[:, t][:, grp]                                                      # [B, H, N]
        Ct = Cm[:, t][:, grp]
        h = dA[:, :, None, None] * h + (dt[:, t][:, :, None] * x[:, t])[..., None] * Bt[:, :, None, :]
        y[:, t] = np.einsum("bhpn,bhn->bhp", h, Ct) + Dsk[None, :, None] * x[:, t]
    y = y.reshape(Bsz, L, E)
    g = y * silu(z)
    o = g / np.sqrt(np.mean(g * g, axis=-1, keepdims=True) + m2.eps) * _f64(w["norm_w"])
    return residual + o @ _f64(w["w_out"]).T, (conv_new, h)


def mixer_forward_tp(m2, w, x_in, residual, k):
    """The same block on k ranks (reading M1): rank r owns heads [r H/k, (r+1) H/k); B and C are
    replicated (n_groups == 1); the gated RMSNorm's per-token sum of squares and the out_proj
    partials are summed in rank order (the two all-reduces).  From the zero state; returns out."""
    x_in, residual = _f64(x_in), _f64(residual)
    E, N, P, G = m2.d_inner, m2.d_state, m2.headdim, m2.n_groups
    H = E // P
    assert G == 1 and H % k == 0
    Hk, Ek = H // k, E // k
    conv_dim = E + 2 * G * N
    W = _f64(w["w_in"])
    parts, ss = [], None
    for r in range(k):
        ch = np.arange(r * Ek, (r + 1) * Ek)
        hs = np.arange(r * Hk, (r + 1) * Hk)
        rows = np.concatenate([ch, E + ch, 2 * E + np.arange(2 * G * N), E + conv_dim + hs])
        cidx = np.concatenate([ch, E + np.arange(2 * G * N)])
        wr = {"conv_w": _f64(w["conv_w"])[cidx], "conv_b": _f64(w["conv_b"])[cidx],
              "dt_bias": _f64(w["dt_bias"])[hs], "a_log": _f64(w["a_log"])[hs], "d_skip": _f64(w["d_skip"])[hs]}
        proj = x_in @ W[rows].T
        g = _gated(Ek, N, P, G, m2.d_conv, wr, proj) * silu(proj[..., :Ek])
        s_r = np.sum(g * g, axis=-1, keepdims=True)
        ss = s_r if ss is None else ss + s_r                       # all-reduce 1 (rank order)
        parts.append((g, _f64(w["norm_w"])[ch], _f64(w["w_out"])[:, ch]))
    rs = 1.0 / np.sqrt(ss / E + m2.eps)
    out = None
    for g, nw, wo in parts:
        p = (g * rs * nw) @ wo.T
        out = p if out is None else out + p                        # all-reduce 2 (rank order)
    return residual + out


def _gated(E, N, P, G, K, w, proj):
    """y (before the gate) of a rank-local mixer of E channels from its projection [z | x | B | C |
    dt], zero initial state (helper of mixer_forward_tp; same steps as mixer_forward)."""
    Bsz, L, _ = proj.shape
    H = E // P
    conv_dim = E + 2 * G * N
    xbc = proj[..., E:E + conv_dim]
    dt = proj[..., E + conv_dim:]
    xt = np.concatenate([np.zeros((Bsz, K - 1, conv_dim)), xbc], axis=1)
    cw = _f64(w["conv_w"])
    xc = np.zeros_like(xbc)
    for j in range(K):
        xc += xt[:, j:j + L, :] * cw[:, j]
    u = silu(xc + _f64(w["conv_b"]))
    x = u[..., :E].reshape(Bsz, L, H, P)
    Bm = u[..., E:E + G * N].reshape(Bsz, L, G, N)
    Cm = u[..., E + G * N:].reshape(Bsz, L, G, N)
    dt = softplus(dt + _f64(w["dt_bias"]))
    A = -np.exp(_f64(w["a_log"]))
    grp = np.arange(H) // (H // G)
    h = np.zeros((Bsz, H, P, N))
    y = np.zeros((Bsz, L, H, P))
    for t in range(L):
        dA = np.exp(dt[:, t] * A)
        h = dA[:, :, None, None] * h + (dt[:, t][:, :, None] * x[:, t])[..., None] * Bm[:, t][:, grp][:, :, None, :]
        y[:, t] = np.einsum("bhpn,bhn->bhp", h, Cm[:, t][:, grp]) + _f64(w["d_skip"])[None, :, None] * x[:, t]
    return y.reshape(Bsz, L, E)
