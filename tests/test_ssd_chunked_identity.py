"""Reading M2: the chunked SSD form that `m2_ssd_chunk_kernel` evaluates equals the
per-token recurrence of the Mamba-2 scan (oracle/mamba2_ref.py mixer_forward's loop)
up to rounding, for ragged chunks, a non-zero carried state and heads sharing one B/C group.

Per chunk of Q tokens, with a_s = dt_s A and the in-chunk inclusive cumulative sum A_t:
    y_t   = exp(A_t) C_t h_prev^T + sum_{s<=t} (C_t . B_s) exp(A_t - A_s) dt_s x_s
    h_end = exp(A_Q) h_prev + sum_s exp(A_Q - A_s) dt_s x_s B_s^T
Both sides in fp64 numpy; no GPU, no product code.
"""
import numpy as np
import pytest


def recurrence(x, Bm, Cm, dt, A, h0):
    """h_t = exp(dt_t A) h_{t-1} + dt_t x_t B_t^T, y_t = h_t C_t (per head; x [L, H, P], B/C [L, N])."""
    L, H, P = x.shape
    h = h0.copy()
    y = np.zeros((L, H, P))
    for t in range(L):
        dA = np.exp(dt[t] * A)                                           # [H]
        h = dA[:, None, None] * h + (dt[t][:, None] * x[t])[..., None] * Bm[t][None, None, :]
        y[t] = h @ Cm[t]
    return y, h


def chunked(x, Bm, Cm, dt, A, h0, Q):
    L, H, P = x.shape
    h = h0.copy()
    y = np.zeros((L, H, P))
    for c0 in range(0, L, Q):
        sl = slice(c0, min(L, c0 + Q))
        xc, Bc, Cc, dc = x[sl], Bm[sl], Cm[sl], dt[sl]                   # [q, H, P], [q, N], [q, N], [q, H]
        q = xc.shape[0]
        Acum = np.cumsum(dc * A[None, :], axis=0)                        # [q, H] inclusive
        G = Cc @ Bc.T                                                    # [q (t), q (s)]
        mask = np.tril(np.ones((q, q)))
        for hd in range(H):
            decay = np.exp((Acum[:, hd][:, None] - Acum[:, hd][None, :]) * mask) * mask
            M = G * decay * dc[:, hd][None, :]                           # (G o decay) dt_s
            y[sl, hd] = np.exp(Acum[:, hd])[:, None] * (Cc @ h[hd].T) + M @ xc[:, hd]
            w = np.exp(Acum[-1, hd] - Acum[:, hd]) * dc[:, hd]           # [q]
            h[hd] = np.exp(Acum[-1, hd]) * h[hd] + (xc[:, hd] * w[:, None]).T @ Bc
    return y, h


@pytest.mark.parametrize("L,Q", [(150, 64), (64, 64), (17, 64), (130, 16)])
def test_chunked_ssd_equals_recurrence(L, Q):
    rng = np.random.default_rng(L * 31 + Q)
    H, P, N = 3, 8, 16
    x = rng.standard_normal((L, H, P))
    Bm = rng.standard_normal((L, N))
    Cm = rng.standard_normal((L, N))
    dt = np.log1p(np.exp(rng.standard_normal((L, H)) - 1.0))            # softplus: dt > 0
    A = -np.exp(rng.uniform(-1.0, 1.0, H))
    h0 = rng.standard_normal((H, P, N))
    y_ref, h_ref = recurrence(x, Bm, Cm, dt, A, h0)
    y, h = chunked(x, Bm, Cm, dt, A, h0, Q)
    np.testing.assert_allclose(y, y_ref, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(h, h_ref, rtol=1e-10, atol=1e-10)


def test_chunked_ssd_strong_decay_underflows_cleanly():
    """dt A of -60 per token: in-chunk decays reach exp(-3800); masked entries never form exp(+x)."""
    L, H, P, N = 80, 2, 4, 8
    rng = np.random.default_rng(7)
    x = rng.standard_normal((L, H, P))
    Bm, Cm = rng.standard_normal((L, N)), rng.standard_normal((L, N))
    dt = np.full((L, H), 3.0)
    A = np.array([-20.0, -0.01])
    h0 = rng.standard_normal((H, P, N))
    y_ref, h_ref = recurrence(x, Bm, Cm, dt, A, h0)
    with np.errstate(over="raise"):
        y, h = chunked(x, Bm, Cm, dt, A, h0, 64)
    assert np.all(np.isfinite(y))
    np.testing.assert_allclose(y, y_ref, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(h, h_ref, rtol=1e-9, atol=1e-9)
