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
