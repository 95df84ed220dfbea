"""Pins of the TP simulation (§4.2-4.3) and the int8 quantised
all-reduce (§4.4; north_star int8 reading)."""
import os

import numpy as np
import pytest

import synth
from oracle import mixer_ref as M
from oracle import qar_ref as Q
from oracle import tp_sim as T

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _tiny(**kw):
    base = dict(d_model=64, d_inner=128, d_state=16, d_conv=4, dt_rank=4, n_layers=1)
    base.update(kw)
    return synth.MixerDims(**base)


def _np(w):
    return {k: v.numpy() for k, v in w.items()}


def test_shard_index_examples():
    # d_inner=4, P=2, r=1 -> W_in rows {2,3} u {6,7}
    assert T.in_proj_rows(4, 2, 1) == [2, 3, 6, 7]
    # d_inner=128, P=4, r=2 -> [64, 96)
    assert T.channel_range(128, 4, 2) == (64, 96)
    with pytest.raises(T.ShardError):
        T.channel_range(100, 3, 0)
    with pytest.raises(T.RankError):
        T.channel_range(128, 4, 4)


def test_shards_reassemble_bitwise():
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    for k in (1, 2, 4):
        sh = [T.shard_weights(dims, w, k, r) for r in range(k)]
        np.testing.assert_array_equal(np.concatenate([s["w_out"] for s in sh], 1), w["w_out"])
        np.testing.assert_array_equal(np.concatenate([s["a_log"] for s in sh], 0), w["a_log"])
        E = dims.d_inner
        xs = np.concatenate([s["w_in"][: E // k] for s in sh], 0)
        zs = np.concatenate([s["w_in"][E // k:] for s in sh], 0)
        np.testing.assert_array_equal(np.concatenate([xs, zs], 0), w["w_in"])
        np.testing.assert_array_equal(np.concatenate([s["heads"][0][2] for s in sh], 1), w["w_x"][0])


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_tp_equals_single_rank(k):
    # TP output matches single-rank mixer up to fp64 reassociation; k=1 bitwise
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, 16, dims.d_model, seed=21)
    ref, st_ref = M.mixer_forward(dims, w, x.numpy(), res.numpy())
    outs, sts, stats = T.tp_mixer_forward(dims, w, x.numpy(), res.numpy(), k)
    for o in outs:
        if k == 1:
            np.testing.assert_array_equal(o, ref)
        else:
            assert np.abs(o - ref).max() / np.abs(ref).max() < 1e-13
    g = T.gather_state(sts)
    np.testing.assert_allclose(g[1], st_ref[1], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(g[0], st_ref[0], rtol=1e-13, atol=1e-14)
    # exactly two all-reduces per block (k>1), none at k=1 (Q13)
    assert stats["allreduce"] == (2 if k > 1 else 0)
    assert stats["allgather"] == 0


@pytest.mark.parametrize("k", [1, 2, 4])
def test_tp_zamba_heads(k):
    dims = _tiny(n_heads=2)
    w = _np(synth.layer_weights(dims, 3))
    x, res = synth.activations(2, 9, dims.d_model, seed=22)
    ref, _ = M.mixer_forward(dims, w, x.numpy(), res.numpy())
    outs, _, stats = T.tp_mixer_forward(dims, w, x.numpy(), res.numpy(), k)
    assert np.abs(outs[0] - ref).max() / np.abs(ref).max() < 1e-13
    # Q17: head-aligned shards at k=2 need no AR#1
    assert stats["allreduce"] == {1: 0, 2: 1, 4: 2}[k]


def test_tp_prefill_decode_cache_equivalence():
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, 12, dims.d_model, seed=23)
    x, res = x.numpy(), res.numpy()
    k = 4
    full, _, _ = T.tp_mixer_forward(dims, w, x, res, k)
    o, st, _ = T.tp_mixer_forward(dims, w, x[:, :9], res[:, :9], k)
    outs = [o[0]]
    for t in range(9, 12):
        o, st, _ = T.tp_mixer_forward(dims, w, x[:, t:t + 1], res[:, t:t + 1], k, states=st)
        outs.append(o[0])
    np.testing.assert_allclose(np.concatenate(outs, 1), full[0], rtol=1e-12, atol=1e-12)


def test_qar_golden_block():
    vals = {}
    with open(os.path.join(GOLD, "qar_block.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                key, *rest = line.split()
                vals[key] = rest
    block = int(vals["block"][0])
    o = np.array(vals["input"], np.float32)[None, :]
    q, s = Q.quantize_blocks(o, block)
    assert s[0, 0] == np.float32(vals["scale"][0])
    np.testing.assert_array_equal(q[0], np.array(vals["codes"], np.int8))
    d = Q.dequantize_blocks(q, s, block)
    np.testing.assert_array_equal(d[0], np.array(vals["dequant"], float))
    err = np.abs(d - o)
    np.testing.assert_array_equal(err[0, 1:], [s[0, 0] / 2] * 3)   # the bound is tight


def test_qar_invariants():
    rng = np.random.default_rng(31)
    # amax -> code +-127 exactly; zero block -> zero scale and codes; never -128
    o = rng.standard_normal((5, 256)).astype(np.float32)
    o[2, :128] = 0
    q, s = Q.quantize_blocks(o, 128)
    assert q.min() >= -127 and q.max() <= 127
    assert s[2, 0] == 0 and np.all(q[2, :128] == 0)
    for r in (0, 1, 3):
        for b in range(2):
            blk = o[r, b * 128:(b + 1) * 128]
            i = np.argmax(np.abs(blk))
            assert abs(int(q[r, b * 128 + i])) == 127
    # exactly representable: values that are integer multiples of s are reproduced exactly
    base = (rng.integers(-127, 128, (1, 128))).astype(np.float32) * np.float32(0.25)
    base[0, 0] = 127 * 0.25
    q, s = Q.quantize_blocks(base, 128)
    np.testing.assert_array_equal(Q.dequantize_blocks(q, s, 128), base)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_qar_error_within_bounds(k):
    parts = synth.partials(k, 8 * 512, seed=40 + k).numpy().reshape(k, 8, 512)
    res, codes, scales = Q.qallreduce(list(parts), 128)
    exact = parts.astype(np.float64).sum(0)
    err = np.abs(res - exact)
    assert np.all(err <= Q.error_bound(scales, 128) * (1 + 1e-12))
    assert np.all(err <= Q.northstar_bound(list(parts), 128) * (1 + 1e-12))


def test_tp_int8_ar2_within_bound():
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, 8, dims.d_model, seed=24)
    k = 2
    ex, _, _ = T.tp_mixer_forward(dims, w, x.numpy(), res.numpy(), k, ar2="exact", block=64)
    q8, _, _ = T.tp_mixer_forward(dims, w, x.numpy(), res.numpy(), k, ar2="int8", block=64)
    d = np.abs(q8[0] - ex[0])
    assert d.max() > 0
    assert d.max() / np.abs(ex[0] - res.numpy()).max() < 2 * k / 254 + 1e-6


# ---------------------------------------------------------------- FP16-wire all-reduce
def _golden_fp16():
    path = os.path.join(os.path.dirname(__file__), "golden", "fp16_cast.txt")
    rows = []
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        a, b = line.split()[:2]
        rows.append((float(a), float(b)))
    return rows


def test_fp16_cast_golden():
    """Hand-derived binary16 RNE cases (ties to even, overflow midpoint, subnormal ties)."""
    import warnings
    for a, b in _golden_fp16():
        assert np.float32(a) == a, "golden inputs are exact fp32 values"
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            got = float(Q.fp16_cast(np.array([a], dtype=np.float32))[0])
        assert got == b, (a, got, b)


def test_fp16_cast_matches_torch_half():
    """A second library's IEEE cast (torch CPU .half()) agrees element for element."""
    import torch
    rng = np.random.default_rng(5)
    o = (rng.standard_normal(4096) * np.exp(rng.uniform(-20, 10, 4096))).astype(np.float32)
    ref = torch.from_numpy(o).half().float().numpy()
    np.testing.assert_array_equal(Q.fp16_cast(o).astype(np.float32), ref)


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_fp16_allreduce_exact_when_representable(k):
    """Partials that are fp16-exact with an fp32-exact sum: the result is the exact sum."""
    rng = np.random.default_rng(k)
    parts = [(rng.integers(-2048, 2048, 512) * 2.0 ** -10).astype(np.float32) for _ in range(k)]
    got, wire = Q.fp16_allreduce(parts)
    exact = np.sum([p.astype(np.float64) for p in parts], axis=0)
    np.testing.assert_array_equal(got.astype(np.float64), exact)
    for w, p in zip(wire, parts):
        np.testing.assert_array_equal(w.astype(np.float32), p)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_fp16_allreduce_within_bound(k):
    rng = np.random.default_rng(100 + k)
    parts = [(rng.standard_normal(8192) * np.exp(rng.uniform(-12, 4, 8192))).astype(np.float32) for _ in range(k)]
    got, _ = Q.fp16_allreduce(parts)
    exact = np.sum([p.astype(np.float64) for p in parts], axis=0)
    err = np.abs(got.astype(np.float64) - exact)
    bound = Q.fp16_error_bound(parts)
    assert np.all(err <= bound)
    assert np.max(err / bound) > 0.25  # the bound is not vacuous


def test_fp16_allreduce_rank_order_and_k1():
    """k = 1 is the cast itself; the fp32 reduction runs left to right in rank order."""
    o = np.array([1.00146484375, 0.1, -3.0], dtype=np.float32)
    got, _ = Q.fp16_allreduce([o])
    np.testing.assert_array_equal(got, np.array([1.001953125, 0.0999755859375, -3.0], dtype=np.float32))
    # 2048 + 2^-13 + 2^-13 in fp32 (ulp(2048) = 2^-12): left to right each add is a tie that
    # rounds to even (2048) -- the order is part of the definition; (b + b) + a would be exact
    a = np.array([2048.0], dtype=np.float32)          # fp16-exact
    b = np.array([2 ** -13], dtype=np.float32)        # fp16-exact (normal)
    got, _ = Q.fp16_allreduce([a, b, b])
    assert got[0] == np.float32(2048.0)
    got, _ = Q.fp16_allreduce([b, b, a])
    assert got[0] == np.float32(2048.0 + 2 ** -12)


def test_tp_fp16_ar2_within_bound():
    """TP=2 mixer with the paper's fp16 AR#2 stays within the fp16 bound of the exact TP result."""
    dims = synth.CONFIGS["tiny"]
    w = {k_: v.numpy() for k_, v in synth.layer_weights(dims, 0).items()}
    x, res = synth.activations(2, 16, dims.d_model)
    x, res = x.numpy(), res.numpy()
    exact, _, _ = T.tp_mixer_forward(dims, w, x, res, 2, ar2="exact")
    f16, _, _ = T.tp_mixer_forward(dims, w, x, res, 2, ar2="fp16")
    d = np.abs(f16[0] - exact[0])
    assert d.max() > 0  # it did quantise
    assert d.max() <= 2 * 2.0 ** -11 * np.abs(exact[0] - res).max() + 1e-6


# ---------------------------------------------------------------- two-shot shared-scale int8 (Q6)
def test_twoshot_golden():
    rows = [list(map(float, l.split())) for l in open(os.path.join(os.path.dirname(__file__), "golden", "qar_twoshot.txt"))
            if l.strip() and not l.startswith("#")]
    o0, o1, want, wantQ = (np.array(r, dtype=np.float32) for r in rows)
    out, codes, s = Q.qallreduce_twoshot([o0, o1], 4)
    assert float(s[0]) == 0.0625
    np.testing.assert_array_equal(codes[0].astype(np.int64) + codes[1].astype(np.int64), wantQ.astype(np.int64))
    np.testing.assert_array_equal(out, want)


def test_twoshot_k1_equals_oneshot():
    """k = 1: the shared scale is the rank's own scale, so the codes equal the one-shot codes."""
    rng = np.random.default_rng(11)
    o = (rng.standard_normal(1024) * np.exp(rng.uniform(-3, 3, 1024))).astype(np.float32)
    out, codes, s = Q.qallreduce_twoshot([o], 128)
    q1, s1 = Q.quantize_blocks(o, 128)
    np.testing.assert_array_equal(codes[0], q1)
    np.testing.assert_array_equal(s, s1)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_twoshot_within_northstar_bound(k):
    rng = np.random.default_rng(40 + k)
    parts = [(rng.standard_normal(4096) * np.exp(rng.uniform(-2, 2, 4096))).astype(np.float32) for _ in range(k)]
    out, codes, s = Q.qallreduce_twoshot(parts, 128)
    exact = np.sum([p.astype(np.float64) for p in parts], axis=0)
    err = np.abs(out.astype(np.float64) - exact)
    bound = Q.northstar_bound(parts, 128)
    assert np.all(err <= bound * (1 + 1e-6) + 1e-30)
    assert np.max(err / bound) > 0.2                 # not vacuous
    for q in codes:
        assert q.min() >= -127 and q.max() <= 127


def _bounds_golden():
    vals = {}
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "qar_bounds.txt")):
        if line.strip() and not line.startswith("#"):
            key, *rest = line.split()
            vals[key] = [float(v) for v in rest]
    return vals


def test_northstar_bound_golden():
    """northstar_bound = k max_r amax / 254 exactly on the hand-worked blocks (a bound constant of
    127, a missing k or a mean instead of a max fails)."""
    g = _bounds_golden()
    rows = [np.array(list(map(float, l.split())), np.float32)
            for l in open(os.path.join(os.path.dirname(__file__), "golden", "qar_twoshot.txt"))
            if l.strip() and not l.startswith("#")]
    b2 = Q.northstar_bound([rows[0], rows[1]], 4)
    np.testing.assert_array_equal(b2, np.full(4, g["northstar_k2"][0]))
    o = np.array([7.9375, 0.03125, -0.09375, 0.15625], np.float32)
    b1 = Q.northstar_bound([o], 4)
    np.testing.assert_array_equal(b1, np.full(4, g["northstar_k1"][0]))
    q, s = Q.quantize_blocks(o[None], 4)
    np.testing.assert_array_equal(Q.error_bound([s], 4)[0], b1)        # = s / 2 here
    err = np.abs(Q.dequantize_blocks(q, s, 4)[0] - o)
    assert np.sum(err == b1) == 3                                      # attained (tight)


def test_fp16_error_bound_golden():
    g = _bounds_golden()
    want = sum(2.0 ** e for e in g["fp16_k2_exponents"])
    got = Q.fp16_error_bound([np.array([1.0], np.float32), np.array([3.0], np.float32)])
    assert got[0] == want
    o = np.array(g["fp16_tie_input"], np.float32)
    got, _ = Q.fp16_allreduce([o])
    err = abs(float(got[0]) - float(o[0]))
    assert err == g["fp16_tie_error"][0]
    assert err <= Q.fp16_error_bound([o])[0] <= err * (1 + 2.0 ** -10)   # attained up to 2^-25


# ---------------------------------------------------------------- bf16-wire all-reduce (custom bf16 arm)
def test_bf16_cast_golden():
    """Hand-derived bfloat16 RNE cases (ties to even at several exponents)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "bf16_cast.txt")
    n = 0
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        a, b = (float(v) for v in line.split()[:2])
        got = float(Q.bf16_cast(np.array([a], dtype=np.float32))[0])
        assert got == b, (a, got, b)
        n += 1
    assert n == 8


def test_bf16_cast_matches_torch_bfloat16():
    """A second library's cast (torch CPU .bfloat16()) agrees element for element."""
    import torch
    rng = np.random.default_rng(6)
    o = (rng.standard_normal(8192) * np.exp(rng.uniform(-40, 40, 8192))).astype(np.float32)
    ref = torch.from_numpy(o).bfloat16().float().numpy()
    np.testing.assert_array_equal(Q.bf16_cast(o), ref)


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_bf16_allreduce_exact_and_bound(k):
    rng = np.random.default_rng(200 + k)
    parts = [(rng.integers(-128, 128, 512) * 2.0 ** -6).astype(np.float32) for _ in range(k)]
    got, wire = Q.bf16_allreduce(parts)                      # bf16-exact partials, exact sums
    np.testing.assert_array_equal(got.astype(np.float64), np.sum([p.astype(np.float64) for p in parts], axis=0))
    parts = [(rng.standard_normal(8192) * np.exp(rng.uniform(-8, 8, 8192))).astype(np.float32) for _ in range(k)]
    got, _ = Q.bf16_allreduce(parts)
    exact = np.sum([p.astype(np.float64) for p in parts], axis=0)
    err = np.abs(got.astype(np.float64) - exact)
    bound = Q.bf16_error_bound(parts)
    assert np.all(err <= bound)
    assert np.max(err / bound) > 0.25                        # not vacuous


def test_tp_bf16_ar2_within_bound():
    dims = synth.CONFIGS["tiny"]
    w = {k_: v.numpy() for k_, v in synth.layer_weights(dims, 0).items()}
    x, res = synth.activations(2, 16, dims.d_model)
    x, res = x.numpy(), res.numpy()
    exact, _, _ = T.tp_mixer_forward(dims, w, x, res, 2, ar2="exact")
    b16, _, _ = T.tp_mixer_forward(dims, w, x, res, 2, ar2="bf16")
    d = np.abs(b16[0] - exact[0])
    assert d.max() > 0
    assert d.max() <= 2 * 2.0 ** -8 * np.abs(exact[0] - res).max() + 1e-6


# ---------------------------------------------------------------- naive 4-collective baseline (§4.2)
@pytest.mark.parametrize("k", [2, 4])
def test_naive_tp_four_collectives_equals_single_rank(k):
    """PAPER.md:297 ("can grow to four per block"), 306 ("lowers the required AllReduces from four
    (under naive sharding) to two"): the naive arm computes the same block with 2 all-gathers + 2
    all-reduces, moving strictly more data than the channel splitter's 2 all-reduces."""
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, 12, dims.d_model, seed=9)
    ref, st_ref = M.mixer_forward(dims, w, x.numpy(), res.numpy())
    outs, sts, st = T.tp_mixer_forward_naive(dims, w, x.numpy(), res.numpy(), k)
    np.testing.assert_allclose(outs[0], ref, rtol=1e-12, atol=1e-12)
    assert st["allgather"] == 2 and st["allreduce"] == 2
    h = T.gather_state(sts)[1]
    np.testing.assert_allclose(h, st_ref[1], rtol=1e-12, atol=1e-12)
    _, _, st_opt = T.tp_mixer_forward(dims, w, x.numpy(), res.numpy(), k)
    assert st_opt["allreduce"] == 2 and st_opt["allgather"] == 0
    opt_elems = 2 * 12 * (dims.dt_rank + 2 * dims.d_state + dims.d_model)
    assert st["elements"] > opt_elems
    # the naive arm's in_proj split straddles the packed field boundary for every k (its rank 0 owns
    # x rows only when k = 2, x and z rows of different channels otherwise) -- the §4.3 pitfall
    wn = 2 * dims.d_inner // k
    assert set(range(0, wn)) != set(T.in_proj_rows(dims.d_inner, k, 0))


# ---------------------------------------------------------------- requantised two-shot (labelled variant)
def test_requant_golden():
    rows = [list(map(float, l.split())) for l in open(os.path.join(os.path.dirname(__file__), "golden", "qar_requant.txt"))
            if l.strip() and not l.startswith("#")]
    o0, o1 = (np.array(r, dtype=np.float32) for r in rows[:2])
    out, codes, scales, q2, s2 = Q.qallreduce_requant([o0, o1], 4)
    np.testing.assert_array_equal(q2.astype(np.int64), np.array(rows[2], dtype=np.int64))
    np.testing.assert_array_equal(out, np.array(rows[3], dtype=np.float32))
    assert float(s2[0]) == rows[4][0]
    np.testing.assert_array_equal(codes[1], np.array([127, 16, 1, -3], np.int8))


def test_requant_k1_reproduces_oneshot():
    """k = 1: the dequantised codes are multiples of s with the block maximum at 127 s, so the
    requantisation returns the same codes and scale."""
    rng = np.random.default_rng(12)
    o = (rng.standard_normal(2048) * np.exp(rng.uniform(-3, 3, 2048))).astype(np.float32)
    out, codes, scales, q2, s2 = Q.qallreduce_requant([o], 128)
    np.testing.assert_array_equal(q2, codes[0])
    np.testing.assert_array_equal(s2, scales[0])


@pytest.mark.parametrize("k", [2, 4, 8])
def test_requant_within_twice_northstar_bound(k):
    rng = np.random.default_rng(70 + k)
    parts = [(rng.standard_normal(4096) * np.exp(rng.uniform(-2, 2, 4096))).astype(np.float32) for _ in range(k)]
    out, *_ = Q.qallreduce_requant(parts, 128)
    exact = np.sum([p.astype(np.float64) for p in parts], axis=0)
    err = np.abs(out.astype(np.float64) - exact)
    bound = 2 * Q.northstar_bound(parts, 128)
    assert np.all(err <= bound * (1 + 1e-6))
    assert np.max(err / Q.northstar_bound(parts, 128)) > 0.5       # the second rounding shows
