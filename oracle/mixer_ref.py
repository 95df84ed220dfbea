"""Single-rank Mamba mixer oracle, numpy float64 (TEST INFRASTRUCTURE ONLY).

Follows the execution order of PAPER.md:151-174 (§2.2, fig:mamba_mixer_block):
input projection -> split (SSM path x, gate path z) -> short causal depthwise
conv -> SSM-parameter projection -> split into dt, B, C -> discretisation ->
sequential state update -> gate -> output projection -> residual add.
Conventions the paper leaves open follow SPEC.md and SURVEY.md §8(c) Q1-Q20
(listed in DESIGN.md §Readings).

Shapes: x_in/residual [B, L, D]; weights as synth.layer_weights documents;
state = (conv_state [B, E, K-1], h [B, E, N]).
"""
from __future__ import annotations

import numpy as np


def _f64(a):
    return np.asarray(a, dtype=np.float64)


# ---------------------------------------------------------------- elementwise
def softplus(v):
    """softplus(v) = ln(1+e^v), linear above 20."""
    v = _f64(v)
    out = np.empty_like(v)
    big = v > 20.0
    out[big] = v[big]
    out[~big] = np.log1p(np.exp(v[~big]))
    return out


def silu(v):
    """SiLU(v) = v * sigmoid(v) (Q2)."""
    v = _f64(v)
    return v / (1.0 + np.exp(-v))


def rmsnorm(x, weight=None, eps=1e-5):
    """x / sqrt(mean(x^2) + eps) * weight over the last axis (pre-norm glue, Q16;
    weightless form with eps=1e-6 is Falcon's dt/B/C norm, Q18)."""
    x = _f64(x)
    r = x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return r if weight is None else r * _f64(weight)


# ---------------------------------------------------------------- sub-ops
def in_proj(x_in, w_in):
    """Packed input projection and split:
    xz = x_in @ w_in^T; x = xz[..., :E] (SSM path), z = xz[..., E:] (gate)."""
    xz = _f64(x_in) @ _f64(w_in).T
    E = xz.shape[-1] // 2
    return xz[..., :E], xz[..., E:]


def causal_conv1d(x, conv_w, conv_b, conv_state=None):
    """Channel-separable causal conv over time.

    x [B, L, E]; conv_w [E, K]; conv_b [E]; conv_state [B, E, K-1] (the last
    K-1 raw inputs before x, zeros at sequence start).
      xt = concat(conv_state, x) along time                (length K-1+L)
      y[b,t,d] = conv_b[d] + sum_j conv_w[d,j] * xt[b, t+j, d]   (tap K-1 = current token)
      conv_state' = last K-1 entries of xt
    Returns (y [B, L, E], conv_state' [B, E, K-1]).  No activation here.
    """
    x = _f64(x)
    Bsz, L, E = x.shape
    K = conv_w.shape[1]
    if conv_state is None:
        conv_state = np.zeros((Bsz, E, K - 1))
    xt = np.concatenate([np.transpose(_f64(conv_state), (0, 2, 1)), x], axis=1)  # [B, K-1+L, E]
    y = np.zeros((Bsz, L, E)) + _f64(conv_b)[None, None, :]
    for j in range(K):
        y = y + _f64(conv_w)[None, None, :, j] * xt[:, j:j + L, :]
    new_state = np.transpose(xt[:, xt.shape[1] - (K - 1):, :], (0, 2, 1)).copy()
    return y, new_state


def split_ssm_params(dbc, dt_rank, d_state):
    """Split the packed SSM-parameter tensor by column range (
    SPEC.md:155): [0,R) -> dt input, [R,R+N) -> B, [R+N,R+2N) -> C."""
    R, N = dt_rank, d_state
    return dbc[..., :R], dbc[..., R:R + N], dbc[..., R + N:R + 2 * N]


def discretize(delta_t, A, B_t):
    """ZOH for A, Euler for B ("scales B accordingly"):
    A_bar[b,d,n] = exp(delta_t[b,d] * A[d,n]);  Bu_factor[b,d,n] = delta_t[b,d] * B_t[b,n]."""
    delta_t, A, B_t = _f64(delta_t), _f64(A), _f64(B_t)
    A_bar = np.exp(delta_t[:, :, None] * A[None, :, :])
    B_bar = delta_t[:, :, None] * B_t[:, None, :]
    return A_bar, B_bar


def scan_step(u_t, delta_t, A, B_t, C_t, D, h):
    """One state update:
    h' = A_bar * h + B_bar * u_t ;  y_t = <C_t, h'> + D * u_t   (h AFTER the update).
    u_t, delta_t [B, E]; A [E, N]; B_t, C_t [B, N]; D [E]; h [B, E, N]."""
    A_bar, B_bar = discretize(delta_t, A, B_t)
    h_new = A_bar * _f64(h) + B_bar * _f64(u_t)[:, :, None]
    y = np.einsum("ben,bn->be", h_new, _f64(C_t)) + _f64(D)[None, :] * _f64(u_t)
    return y, h_new


def scan_full(u, delta, A, B, C, D, h0):
    """Literal sequential fold of scan_step over t = 0..L-1 (C9).
    u, delta [B, L, E]; B, C [B, L, N]; returns (y [B, L, E], h_L [B, E, N])."""
    u, delta = _f64(u), _f64(delta)
    Bsz, L, E = u.shape
    y = np.zeros((Bsz, L, E))
    h = _f64(h0).copy()
    for t in range(L):
        y[:, t, :], h = scan_step(u[:, t, :], delta[:, t, :], A, B[:, t, :], C[:, t, :], D, h)
    return y, h


# ---------------------------------------------------------------- mixer
def zero_state(batch, d_inner, d_state, d_conv):
    return np.zeros((batch, d_inner, d_conv - 1)), np.zeros((batch, d_inner, d_state))


def mixer_forward(dims, w, x_in, residual, state=None):
    """One mixer layer over a chunk of L tokens, carrying the SSM cache.

    dims: synth.MixerDims; w: dict of float64 arrays (synth.layer_weights);
    x_in [B, L, D] (the block input after the pre-norm); residual [B, L, D];
    state: (conv_state [B,E,K-1], h [B,E,N]) or None for zeros.
    Returns (out = residual + mixer(x_in) [B, L, D], (conv_state', h')).

    Steps (SURVEY.md §8(c) algorithm):
      1 xz = x_in W_in^T ; x, z split
      2 u = SiLU(causal_conv(x))                      (Q2/C6)
      3 per head h: dbc_h = u[:, :, ch_h] W_x[h]^T ; dt_low, B, C split
        (Falcon: weightless RMSNorm, eps=rms_eps, on each field, Q18)
      4 delta = softplus(dt_low W_dt[ch_h]^T + b_dt[ch_h])
      5 A = -exp(A_log); sequential scan with D skip
      6 g = y * SiLU(z)
      7 out = residual + g W_out^T
    """
    w = {k: _f64(v) for k, v in w.items()}
    x_in, residual = _f64(x_in), _f64(residual)
    Bsz, L, _ = x_in.shape
    E, N, K, R, H = dims.d_inner, dims.d_state, dims.d_conv, dims.dt_rank, dims.n_heads
    if state is None:
        state = zero_state(Bsz, E, N, K)
    conv_state, h = state

    x, z = in_proj(x_in, w["w_in"])
    xc, conv_state_new = causal_conv1d(x, w["conv_w"], w["conv_b"], conv_state)
    u = silu(xc)

    A = -np.exp(w["a_log"])
    Eh = E // H
    y = np.zeros((Bsz, L, E))
    h_new = np.zeros_like(_f64(h))
    for hd in range(H):
        ch = slice(hd * Eh, (hd + 1) * Eh)
        dbc = u[:, :, ch] @ w["w_x"][hd].T                    # [B, L, P]
        dt_low, Bm, Cm = split_ssm_params(dbc, R, N)
        if dims.bcdt_rmsnorm:
            dt_low = rmsnorm(dt_low, eps=dims.rms_eps)
            Bm = rmsnorm(Bm, eps=dims.rms_eps)
            Cm = rmsnorm(Cm, eps=dims.rms_eps)
        delta = softplus(dt_low @ w["w_dt"][ch].T + w["b_dt"][ch])
        y[:, :, ch], h_new[:, ch, :] = scan_full(u[:, :, ch], delta, A[ch], Bm, Cm,
                                                 w["d_skip"][ch], _f64(h)[:, ch, :])
    g = y * silu(z)
    out = residual + g @ w["w_out"].T
    return out, (conv_state_new, h_new)


def mixer_prefill(dims, w, x_in, residual, state=None):
    """Prefill = mixer_forward from the zero cache (or a carried one); §4.1."""
    return mixer_forward(dims, w, x_in, residual, state)


def mixer_decode(dims, w, x_t, residual_t, state):
    """Decode = the same pipeline with L=1 seeded from the cache."""
    assert x_t.shape[1] == 1
    return mixer_forward(dims, w, x_t, residual_t, state)


def model_forward(dims, layers, x_tokens_resid, states=None, norm_eps=1e-5):
    """Pre-norm stack (Q16): for each layer, residual += mixer(RMSNorm(residual)).
    layers: list of weight dicts; x_tokens_resid [B, L, D] is the incoming residual.
    Returns (residual_out, states)."""
    res = _f64(x_tokens_resid)
    new_states = []
    for i, w in enumerate(layers):
        st = None if states is None else states[i]
        x_in = rmsnorm(res, None, norm_eps)
        res, st2 = mixer_forward(dims, w, x_in, res, st)
        new_states.append(st2)
    return res, new_states
