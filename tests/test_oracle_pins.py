"""Pins of the oracle's sub-operations against things other than itself:
closed forms printed in SPEC.md, library routines (scipy lfilter, torch conv1d)
on special cases, and a pure-Python brute force on tiny inputs."""
import math
import os

import numpy as np
import pytest
import scipy.signal
import torch

from oracle import mixer_ref as M

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_lines(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.strip() for l in f if l.strip() and not l.startswith("#")]


def test_spec_discretize_examples():
    # SPEC.md:103-104 worked examples
    for line in _golden_lines("spec_scan_examples.txt"):
        if not line.startswith("discretize"):
            continue
        lhs, rhs = line[len("discretize"):].split("->")
        dt, arow, b = [np.array(x.split(), float) for x in lhs.split("|")]
        abar_exp, bu_exp = [np.array(x.split(), float) for x in rhs.split("|")]
        abar, bu = M.discretize(dt.reshape(1, 1), arow.reshape(1, -1), b.reshape(1, -1))
        np.testing.assert_allclose(abar[0, 0], abar_exp, rtol=1e-15)
        np.testing.assert_allclose(bu[0, 0], np.broadcast_to(bu_exp, abar_exp.shape), rtol=1e-15)


def test_spec_zero_step_freezes_state():
    # dt -> 0+ leaves the state unchanged and y = D*u
    h = np.array([[[0.3, -0.7]]])
    y, h2 = M.scan_step(np.array([[2.0]]), np.array([[1e-30]]), np.array([[-1.0, -2.0]]),
                        np.array([[1.0, 1.0]]), np.array([[1.0, 1.0]]), np.array([0.5]), h)
    np.testing.assert_allclose(h2, h, rtol=1e-14)
    np.testing.assert_allclose(y, [[h.sum() + 1.0]], rtol=1e-14)


def test_spec_scan_step_examples():
    gold = {l.split()[0]: [float(v) for v in l.split()[1:]] for l in _golden_lines("spec_scan_examples.txt")
            if l.startswith("step")}
    A = np.array([[-1.0]]); Bt = np.array([[1.0]]); Ct = np.array([[1.0]]); D = np.array([0.0])
    dt = np.array([[math.log(2.0)]])
    y1, h1 = M.scan_step(np.array([[1.0]]), dt, A, Bt, Ct, D, np.zeros((1, 1, 1)))
    assert h1[0, 0, 0] == pytest.approx(gold["step1"][0], rel=1e-15)
    assert y1[0, 0] == pytest.approx(gold["step1"][1], rel=1e-15)
    y2, h2 = M.scan_step(np.array([[0.0]]), dt, A, Bt, Ct, D, h1)
    assert h2[0, 0, 0] == pytest.approx(gold["step2"][0], rel=1e-15)
    assert y2[0, 0] == pytest.approx(gold["step2"][1], rel=1e-15)


def test_softplus_silu_closed_forms():
    gold = {l.split()[0]: float(l.split()[1]) for l in _golden_lines("spec_scan_examples.txt") if l.startswith("softplus0")}
    assert M.softplus(np.array([0.0]))[0] == pytest.approx(gold["softplus0"], rel=1e-15)
    assert M.silu(np.array([0.0]))[0] == 0.0
    # large-argument branch is the identity; continuity at 20
    assert M.softplus(np.array([30.0]))[0] == 30.0
    assert abs(M.softplus(np.array([20.0]))[0] - 20.0) < 3e-9
    # silu(x) - silu(-x) = x  (sigmoid symmetry) -- catches a sign error in the sigmoid
    x = np.linspace(-5, 5, 11)
    np.testing.assert_allclose(M.silu(x) - M.silu(-x), x, atol=1e-14)


def test_scan_constant_params_equals_lfilter():
    """With dt, B, C constant over t, each (d, n) state is a first-order IIR filter:
    h_t = a h_{t-1} + (dt B_n) u_t, a = exp(dt A_dn)  ==  scipy.signal.lfilter([dt*B_n], [1, -a], u)."""
    rng = np.random.default_rng(0)
    Bsz, L, E, N = 2, 40, 3, 5
    u = rng.standard_normal((Bsz, L, E))
    dt_c = rng.uniform(0.01, 0.5, (Bsz, E))
    Bc = rng.standard_normal((Bsz, N))
    Cc = rng.standard_normal((Bsz, N))
    A = -rng.uniform(0.5, 4.0, (E, N))
    Dv = rng.standard_normal(E)
    delta = np.broadcast_to(dt_c[:, None, :], (Bsz, L, E))
    y, hL = M.scan_full(u, delta, A, np.broadcast_to(Bc[:, None, :], (Bsz, L, N)),
                        np.broadcast_to(Cc[:, None, :], (Bsz, L, N)), Dv, np.zeros((Bsz, E, N)))
    for b in range(Bsz):
        for d in range(E):
            ysum = Dv[d] * u[b, :, d]
            for n in range(N):
                a = math.exp(dt_c[b, d] * A[d, n])
                h = scipy.signal.lfilter([dt_c[b, d] * Bc[b, n]], [1.0, -a], u[b, :, d])
                ysum = ysum + Cc[b, n] * h
                assert hL[b, d, n] == pytest.approx(h[-1], rel=1e-12, abs=1e-14)
            np.testing.assert_allclose(y[b, :, d], ysum, rtol=1e-11, atol=1e-13)


def _brute_scan(u, delta, A, Bm, Cm, Dv, h0):
    """Pure-Python scalar loops straight from the two update equations."""
    Bsz, L, E = u.shape
    N = A.shape[1]
    h = [[[h0[b][d][n] for n in range(N)] for d in range(E)] for b in range(Bsz)]
    y = [[[0.0] * E for _ in range(L)] for _ in range(Bsz)]
    for b in range(Bsz):
        for t in range(L):
            for d in range(E):
                acc = 0.0
                for n in range(N):
                    h[b][d][n] = math.exp(delta[b][t][d] * A[d][n]) * h[b][d][n] + delta[b][t][d] * Bm[b][t][n] * u[b][t][d]
                    acc += Cm[b][t][n] * h[b][d][n]
                y[b][t][d] = acc + Dv[d] * u[b][t][d]
    return np.array(y), np.array(h)


def test_scan_full_vs_bruteforce_time_varying():
    # random B=1, L=4, E=2, N=3 instance vs an independent brute-force recurrence
    rng = np.random.default_rng(1)
    for (Bsz, L, E, N) in [(1, 4, 2, 3), (2, 9, 3, 4)]:
        u = rng.standard_normal((Bsz, L, E))
        delta = rng.uniform(0.01, 1.0, (Bsz, L, E))
        A = -np.exp(rng.standard_normal((E, N)))
        Bm = rng.standard_normal((Bsz, L, N)); Cm = rng.standard_normal((Bsz, L, N))
        Dv = rng.standard_normal(E); h0 = rng.standard_normal((Bsz, E, N))
        y, hL = M.scan_full(u, delta, A, Bm, Cm, Dv, h0)
        yb, hb = _brute_scan(u, delta, A, Bm, Cm, Dv, h0)
        np.testing.assert_allclose(y, yb, rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(hL, hb, rtol=1e-13, atol=1e-13)


def test_scan_contraction_zero_input():
    # with u = 0, ||h_t||_inf is non-increasing
    rng = np.random.default_rng(2)
    E, N, L = 4, 6, 20
    A = -np.exp(rng.standard_normal((E, N)))
    h = rng.standard_normal((1, E, N))
    prev = np.abs(h).max()
    for t in range(L):
        _, h = M.scan_step(np.zeros((1, E)), rng.uniform(0.01, 1, (1, E)), A,
                           rng.standard_normal((1, N)), rng.standard_normal((1, N)), np.ones(E), h)
        cur = np.abs(h).max()
        assert cur <= prev + 1e-15
        prev = cur


def test_scan_prefix_consistency_bitwise():
    # split point s; exact (same fp64 ops in the same order)
    rng = np.random.default_rng(3)
    Bsz, L, E, N = 2, 17, 3, 4
    args = (rng.standard_normal((Bsz, L, E)), rng.uniform(0.01, 1, (Bsz, L, E)), -np.exp(rng.standard_normal((E, N))),
            rng.standard_normal((Bsz, L, N)), rng.standard_normal((Bsz, L, N)), rng.standard_normal(E))
    u, dl, A, Bm, Cm, Dv = args
    y, h = M.scan_full(u, dl, A, Bm, Cm, Dv, np.zeros((Bsz, E, N)))
    for s in (0, 1, 8, 16, 17):
        y1, h1 = M.scan_full(u[:, :s], dl[:, :s], A, Bm[:, :s], Cm[:, :s], Dv, np.zeros((Bsz, E, N)))
        y2, h2 = M.scan_full(u[:, s:], dl[:, s:], A, Bm[:, s:], Cm[:, s:], Dv, h1)
        assert np.array_equal(np.concatenate([y1, y2], 1), y)
        assert np.array_equal(h2, h)


def test_conv_identity_and_ones_kernel():
    # SPEC.md:174-175
    x = np.random.default_rng(4).standard_normal((2, 7, 3))
    w = np.zeros((3, 4)); w[:, 3] = 1.0
    y, _ = M.causal_conv1d(x, w, np.zeros(3))
    np.testing.assert_array_equal(y, x)
    y, _ = M.causal_conv1d(np.ones((1, 4, 1)), np.ones((1, 4)), np.zeros(1))
    np.testing.assert_array_equal(y[0, :, 0], [1, 2, 3, 4])


def test_conv_matches_torch_conv1d_and_step_mode():
    # torch.nn.functional.conv1d(groups=E, padding=K-1)[..., :L] is the library form of the
    # channel-separable causal conv ("Conv1d on groups = intermediate_size")
    rng = np.random.default_rng(5)
    Bsz, L, E, K = 2, 11, 6, 4
    x = rng.standard_normal((Bsz, L, E)); w = rng.standard_normal((E, K)); b = rng.standard_normal(E)
    y, st = M.causal_conv1d(x, w, b)
    ref = torch.nn.functional.conv1d(torch.from_numpy(x).transpose(1, 2), torch.from_numpy(w)[:, None, :],
                                     torch.from_numpy(b), padding=K - 1, groups=E)[..., :L]
    np.testing.assert_allclose(y, ref.transpose(1, 2).numpy(), rtol=1e-13, atol=1e-13)
    # state = last K-1 raw inputs
    np.testing.assert_array_equal(st, np.transpose(x[:, L - (K - 1):, :], (0, 2, 1)))
    # SPEC.md:176 step mode: one token at a time with the carried state equals the full output
    state = np.zeros((Bsz, E, K - 1))
    for t in range(L):
        yt, state = M.causal_conv1d(x[:, t:t + 1], w, b, state)
        np.testing.assert_allclose(yt[:, 0], y[:, t], rtol=1e-14, atol=1e-14)
    # short chunk (L < K-1) mixes old state and new input
    s0 = rng.standard_normal((Bsz, E, K - 1))
    _, s1 = M.causal_conv1d(x[:, :2], w, b, s0)
    np.testing.assert_array_equal(s1[:, :, 0], s0[:, :, 2])
    np.testing.assert_array_equal(s1[:, :, 1:], np.transpose(x[:, :2], (0, 2, 1)))


def test_split_round_trips():
    # SPEC.md:165-167, 183-185
    rng = np.random.default_rng(6)
    xz = rng.standard_normal((2, 3, 8))
    w = np.eye(8)
    x, z = M.in_proj(xz, w)
    np.testing.assert_array_equal(np.concatenate([x, z], -1), xz)
    dbc = rng.standard_normal((2, 3, 4 + 2 * 5))
    a, b, c = M.split_ssm_params(dbc, 4, 5)
    np.testing.assert_array_equal(np.concatenate([a, b, c], -1), dbc)
    a, b, c = M.split_ssm_params(np.array([[[7.0, 8.0, 9.0]]]), 1, 1)
    assert (a.item(), b.item(), c.item()) == (7.0, 8.0, 9.0)


def test_rmsnorm_closed_forms():
    x = np.full((1, 8), 3.0)
    np.testing.assert_allclose(M.rmsnorm(x, eps=0.0), np.ones((1, 8)), rtol=1e-15)
    x = np.random.default_rng(7).standard_normal((3, 16))
    # scale invariance (eps=0) and weight multiplies
    np.testing.assert_allclose(M.rmsnorm(5 * x, eps=0.0), M.rmsnorm(x, eps=0.0), rtol=1e-13)
    w = np.arange(16.0)
    np.testing.assert_allclose(M.rmsnorm(x, w, 0.0), M.rmsnorm(x, None, 0.0) * w, rtol=1e-14)
    # mean of squares of the output is 1 (eps=0)
    np.testing.assert_allclose((M.rmsnorm(x, eps=0.0) ** 2).mean(-1), 1.0, rtol=1e-13)
