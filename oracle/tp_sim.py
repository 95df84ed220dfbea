"""Tensor-parallel mixer, ranks simulated in-process (TEST INFRASTRUCTURE ONLY).

Channel splitter (§4.2) and packed-parameter placement
(§4.3) with exactly two all-reduces per block
(PAPER.md:306-311): AR#1 on the SSM-parameter projection, AR#2 at the
residual boundary.  Reduction order is fixed 0..k-1 (Q12).
Readings: A/D row-sharded (C4), B/C taken from AR#1's full vector (C5),
AR#1 unquantised (Q3), AR#2 exact, int8 (qar_ref, Q6-Q9) or the paper's fp16 wire (Q21).
Zamba heads (Q17): channel d belongs to head d // (E/H); AR#1 sums only over
the ranks that own channels of a head.
"""
from __future__ import annotations

import numpy as np

from . import mixer_ref as M
from . import qar_ref


class ShardError(ValueError):
    pass


class RankError(ValueError):
    pass


def channel_range(d_inner, k, r):
    """[lo, hi) owned by rank r."""
    if k < 1 or d_inner % k != 0:
        raise ShardError(f"d_inner={d_inner} not divisible by tp={k}")
    if not 0 <= r < k:
        raise RankError(f"rank {r} not in [0,{k})")
    Ek = d_inner // k
    return r * Ek, (r + 1) * Ek


def in_proj_rows(d_inner, k, r):
    """Global rows of the packed W_in owned by rank r: its x block and its z block
    (SPEC.md:359 example d_inner=4,k=2,r=1 -> {2,3,6,7})."""
    lo, hi = channel_range(d_inner, k, r)
    return list(range(lo, hi)) + list(range(d_inner + lo, d_inner + hi))


def local_heads(dims, k, r):
    """[(head, local channel slice, head-relative column slice)] for rank r."""
    lo, hi = channel_range(dims.d_inner, k, r)
    Eh = dims.d_inner // dims.n_heads
    out = []
    for hd in range(dims.n_heads):
        a, b = max(lo, hd * Eh), min(hi, (hd + 1) * Eh)
        if a < b:
            out.append((hd, slice(a - lo, b - lo), slice(a - hd * Eh, b - hd * Eh)))
    return out


def shard_weights(dims, w, k, r):
    """Rank-local weights (pure slicing, no arithmetic)."""
    lo, hi = channel_range(dims.d_inner, k, r)
    rows = in_proj_rows(dims.d_inner, k, r)
    s = {
        "w_in": np.asarray(w["w_in"])[rows],
        "conv_w": np.asarray(w["conv_w"])[lo:hi],
        "conv_b": np.asarray(w["conv_b"])[lo:hi],
        "w_dt": np.asarray(w["w_dt"])[lo:hi],
        "b_dt": np.asarray(w["b_dt"])[lo:hi],
        "a_log": np.asarray(w["a_log"])[lo:hi],
        "d_skip": np.asarray(w["d_skip"])[lo:hi],
        "w_out": np.asarray(w["w_out"])[:, lo:hi],
        "heads": [],
    }
    for hd, loc, col in local_heads(dims, k, r):
        s["heads"].append((hd, loc, np.asarray(w["w_x"])[hd][:, col]))
    return s


def shard_state(state, d_inner, k, r):
    lo, hi = channel_range(d_inner, k, r)
    conv, h = state
    return conv[:, lo:hi].copy(), h[:, lo:hi].copy()


def gather_state(states):
    return (np.concatenate([s[0] for s in states], axis=1),
            np.concatenate([s[1] for s in states], axis=1))


def tp_mixer_forward(dims, w, x_in, residual, k, states=None, ar2="exact", block=128, stats=None):
    """All k ranks of one TP mixer block, lock-step.

    Returns (outs: list of k [B,L,D] arrays (replicas), states', stats) where
    stats counts collectives with more than one participant.
    """
    x_in, residual = np.asarray(x_in, np.float64), np.asarray(residual, np.float64)
    Bsz, L, _ = x_in.shape
    E, N, K, R = dims.d_inner, dims.d_state, dims.d_conv, dims.dt_rank
    Ek = E // k
    if stats is None:
        stats = {"allreduce": 0, "allgather": 0}
    shards = [shard_weights(dims, w, k, r) for r in range(k)]
    if states is None:
        states = [M.zero_state(Bsz, Ek, N, K) for _ in range(k)]

    # (1)-(3) rank-local in_proj, conv+SiLU, partial x_proj per head
    loc = []
    for r in range(k):
        s = shards[r]
        x, z = M.in_proj(x_in, s["w_in"])
        xc, conv_new = M.causal_conv1d(x, s["conv_w"], s["conv_b"], states[r][0])
        u = M.silu(xc)
        parts = {hd: u[:, :, lc] @ wx.T for hd, lc, wx in s["heads"]}
        loc.append(dict(z=z, u=u, conv=conv_new, parts=parts))

    # AR#1: per head, fixed rank order over the ranks owning that head
    full = {}
    ar1_multi = False
    for hd in range(dims.n_heads):
        owners = [r for r in range(k) if hd in loc[r]["parts"]]
        ar1_multi |= len(owners) > 1
        acc = None
        for r in owners:
            acc = loc[r]["parts"][hd] if acc is None else acc + loc[r]["parts"][hd]
        full[hd] = acc
    if ar1_multi:
        stats["allreduce"] += 1

    # (4)-(7) local unpack, dt_proj, scan, gate, partial out_proj
    partial_out, new_states = [], []
    for r in range(k):
        s, lr = shards[r], loc[r]
        A = -np.exp(s["a_log"])
        y = np.zeros((Bsz, L, Ek))
        h_new = np.zeros((Bsz, Ek, N))
        for hd, lc, _ in s["heads"]:
            dt_low, Bm, Cm = M.split_ssm_params(full[hd], R, N)
            if dims.bcdt_rmsnorm:
                dt_low = M.rmsnorm(dt_low, eps=dims.rms_eps)
                Bm = M.rmsnorm(Bm, eps=dims.rms_eps)
                Cm = M.rmsnorm(Cm, eps=dims.rms_eps)
            delta = M.softplus(dt_low @ s["w_dt"][lc].T + s["b_dt"][lc])
            y[:, :, lc], h_new[:, lc, :] = M.scan_full(lr["u"][:, :, lc], delta, A[lc], Bm, Cm,
                                                       s["d_skip"][lc], states[r][1][:, lc, :])
        g = y * M.silu(lr["z"])
        partial_out.append(g @ s["w_out"].T)
        new_states.append((lr["conv"], h_new))

    # AR#2 at the residual boundary
    if k == 1:
        total = partial_out[0]                     # TP=1: no AR, no quantisation (Q13)
    elif ar2 == "exact":
        total = partial_out[0].copy()
        for r in range(1, k):
            total = total + partial_out[r]
    elif ar2 == "int8":
        total, _, _ = qar_ref.qallreduce([p.astype(np.float32) for p in partial_out], block)
    elif ar2 == "fp16":                            # the paper's FP32 -> FP16 wire
        total, _ = qar_ref.fp16_allreduce([p.astype(np.float32) for p in partial_out])
        total = total.astype(np.float64)
    elif ar2 == "bf16":                            # the custom bf16 wire
        total, _ = qar_ref.bf16_allreduce([p.astype(np.float32) for p in partial_out])
        total = total.astype(np.float64)
    else:
        raise ValueError(ar2)
    if k > 1:
        stats["allreduce"] += 1
    out = residual + total
    return [out.copy() for _ in range(k)], new_states, stats


def tp_mixer_forward_naive(dims, w, x_in, residual, k, states=None, stats=None):
    """The paper's NAIVE sharding baseline (§4.2): "the number of communication
    collectives can grow to four per block because packed intermediate tensors must be repeatedly
    reassembled" -- (i) after the input projection, (ii) around the convolution branch, (iii)
    after the SSM-parameter projection, (iv) when merging the SSM output (the residual boundary).
    Reading N1: W_in is split uniformly along its PACKED first extent (rank r owns
    rows [r 2E/k, (r+1) 2E/k) of [x ; z], straddling the field boundary), so (i) is an all-gather
    of the packed activation; the conv weights follow the channels, so (ii) is an all-gather of the
    conv output back to the full-width layout; (iii) and (iv) are the all-reduces of the channel-
    split design (x_proj and out_proj partials over the rank's channels).  One block, TP = k,
    Mamba/Falcon (one x_proj head).  Returns (outs, states', stats) with stats["allgather"],
    stats["allreduce"] and stats["elements"] (elements each rank contributes, summed over the
    collectives)."""
    x_in, residual = np.asarray(x_in, np.float64), np.asarray(residual, np.float64)
    Bsz, L, D = x_in.shape
    E, N, K, R = dims.d_inner, dims.d_state, dims.d_conv, dims.dt_rank
    assert dims.n_heads == 1 and E % k == 0
    Ek, wn = E // k, 2 * E // k
    if stats is None:
        stats = {"allreduce": 0, "allgather": 0, "elements": 0}
    w_in = np.asarray(w["w_in"])
    if states is None:
        states = [M.zero_state(Bsz, Ek, N, K) for _ in range(k)]
    # (i) uniform slices of the packed in_proj, all-gathered into the full [x ; z]
    xz_parts = [x_in @ w_in[r * wn:(r + 1) * wn].T for r in range(k)]
    xz = np.concatenate(xz_parts, axis=-1)
    stats["allgather"] += 1
    stats["elements"] += Bsz * L * wn
    x_full, z_full = xz[..., :E], xz[..., E:]
    shards = [shard_weights(dims, w, k, r) for r in range(k)]
    # (ii) conv on the owned channels, all-gathered back to the full width
    us, convs = [], []
    for r in range(k):
        s = shards[r]
        xc, conv_new = M.causal_conv1d(x_full[..., r * Ek:(r + 1) * Ek], s["conv_w"], s["conv_b"], states[r][0])
        us.append(M.silu(xc))
        convs.append(conv_new)
    u_full = np.concatenate(us, axis=-1)
    stats["allgather"] += 1
    stats["elements"] += Bsz * L * Ek
    # (iii) x_proj partials over the owned channels of the gathered layout, all-reduced
    wx = np.asarray(w["w_x"])[0]
    dbc = None
    for r in range(k):
        p = u_full[..., r * Ek:(r + 1) * Ek] @ wx[:, r * Ek:(r + 1) * Ek].T
        dbc = p if dbc is None else dbc + p
    stats["allreduce"] += 1
    stats["elements"] += Bsz * L * (R + 2 * N)
    dt_low, Bm, Cm = M.split_ssm_params(dbc, R, N)
    if dims.bcdt_rmsnorm:
        dt_low = M.rmsnorm(dt_low, eps=dims.rms_eps)
        Bm = M.rmsnorm(Bm, eps=dims.rms_eps)
        Cm = M.rmsnorm(Cm, eps=dims.rms_eps)
    # local dt_proj / scan / gate on the owned channels, (iv) out_proj partials all-reduced
    total, new_states = None, []
    for r in range(k):
        s = shards[r]
        delta = M.softplus(dt_low @ s["w_dt"].T + s["b_dt"])
        y, h_new = M.scan_full(us[r], delta, -np.exp(s["a_log"]), Bm, Cm, s["d_skip"], states[r][1])
        g = y * M.silu(z_full[..., r * Ek:(r + 1) * Ek])
        p = g @ s["w_out"].T
        total = p if total is None else total + p
        new_states.append((convs[r], h_new))
    stats["allreduce"] += 1
    stats["elements"] += Bsz * L * D
    out = residual + total
    return [out.copy() for _ in range(k)], new_states, stats
