"""Whole-mixer oracle pins: HF transformers slow paths (float64 on CPU; the
Mamba code lineage whose naming the paper uses), SPEC.md
passthrough examples, and the SSM-cache invariants of PAPER.md §4.1."""
import warnings

import numpy as np
import pytest
import torch

import synth
from oracle import mixer_ref as M


def _tiny(**kw):
    base = dict(d_model=64, d_inner=128, d_state=16, d_conv=4, dt_rank=4, n_layers=1)
    base.update(kw)
    return synth.MixerDims(**base)


def _np(w):
    return {k: v.numpy() for k, v in w.items()}


def _hf_mamba(dims, w, falcon=False):
    warnings.filterwarnings("ignore")
    if falcon:
        from transformers import FalconMambaConfig as Cfg
        from transformers.models.falcon_mamba.modeling_falcon_mamba import FalconMambaMixer as Mixer
    else:
        from transformers import MambaConfig as Cfg
        from transformers.models.mamba.modeling_mamba import MambaMixer as Mixer
    cfg = Cfg(hidden_size=dims.d_model, intermediate_size=dims.d_inner, state_size=dims.d_state,
              conv_kernel=dims.d_conv, time_step_rank=dims.dt_rank, use_bias=False, use_conv_bias=True,
              hidden_act="silu", use_mambapy=False)
    if falcon:
        cfg.mixer_rms_eps = dims.rms_eps
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    try:
        m = Mixer(cfg, layer_idx=0, initialize_mixer_weights=False).eval()
    finally:
        torch.set_default_dtype(prev)
    with torch.no_grad():
        m.in_proj.weight.copy_(w["w_in"])
        m.conv1d.weight.copy_(w["conv_w"][:, None, :])
        m.conv1d.bias.copy_(w["conv_b"])
        m.x_proj.weight.copy_(w["w_x"][0])
        m.dt_proj.weight.copy_(w["w_dt"])
        m.dt_proj.bias.copy_(w["b_dt"])
        m.A_log.copy_(w["a_log"])
        m.D.copy_(w["d_skip"])
        m.out_proj.weight.copy_(w["w_out"])
    return m


def test_mixer_matches_hf_mamba_slow_forward():
    dims = _tiny()
    w = synth.layer_weights(dims, 0)
    x, res = synth.activations(2, 32, dims.d_model)
    m = _hf_mamba(dims, w)
    with torch.no_grad():
        hf = m.slow_forward(x).numpy()
    out, _ = M.mixer_forward(dims, _np(w), x.numpy(), res.numpy())
    mine = out - res.numpy()
    # HF casts A, B, u to fp32 internally (modeling_mamba.py:321-324) -> ~1e-7, not bits
    assert np.abs(mine - hf).max() / np.abs(hf).max() < 2e-6


def test_mixer_matches_hf_falcon_mamba_rmsnorm_variant():
    dims = _tiny(bcdt_rmsnorm=True)
    w = synth.layer_weights(dims, 1)
    x, res = synth.activations(2, 24, dims.d_model, seed=3)
    m = _hf_mamba(dims, w, falcon=True)
    with torch.no_grad():
        hf = m.slow_forward(x).numpy()
    out, _ = M.mixer_forward(dims, _np(w), x.numpy(), res.numpy())
    mine = out - res.numpy()
    assert np.abs(mine - hf).max() / np.abs(hf).max() < 2e-6
    # and the flag matters (the pin would catch a dropped norm)
    out2, _ = M.mixer_forward(_tiny(), _np(w), x.numpy(), res.numpy())
    assert np.abs(out2 - res.numpy() - hf).max() / np.abs(hf).max() > 1e-3


def test_mixer_matches_hf_zamba_two_heads():
    warnings.filterwarnings("ignore")
    from transformers import ZambaConfig
    from transformers.models.zamba.modeling_zamba import ZambaMambaMixer
    dims = _tiny(n_heads=2)
    w = synth.layer_weights(dims, 2)
    cfg = ZambaConfig(hidden_size=dims.d_model, mamba_expand=2, mamba_d_state=dims.d_state,
                      mamba_d_conv=dims.d_conv, mamba_dt_rank=dims.dt_rank, n_mamba_heads=2,
                      mamba_conv_bias=True, mamba_proj_bias=False, hidden_mamba_act="silu",
                      use_mamba_kernels=False, num_hidden_layers=3, attn_layer_period=6,
                      attn_layer_offset=4, num_attention_heads=4, num_key_value_heads=4)
    m = ZambaMambaMixer(cfg, layer_idx=0).double().eval()
    E, H = dims.d_inner, 2
    Eh = E // H
    # Zamba packs in_proj rows interleaved (x_i, z_i) per channel (modeling_zamba.py:372);
    # the build's canonical packing is [x block || z block] -> permute rows to load.
    w_in_hf = torch.empty_like(w["w_in"])
    w_in_hf[0::2] = w["w_in"][:E]
    w_in_hf[1::2] = w["w_in"][E:]
    with torch.no_grad():
        m.in_proj.weight.copy_(w_in_hf)
        m.conv1d.weight.copy_(w["conv_w"][:, None, :])
        m.conv1d.bias.copy_(w["conv_b"])
        m.x_proj_weight.copy_(w["w_x"])
        m.dt_proj_weight.copy_(w["w_dt"].reshape(H, Eh, -1))
        m.dt_proj_bias.copy_(w["b_dt"].reshape(H, Eh))
        m.A_log.copy_(w["a_log"].reshape(H, Eh, -1))
        m.D.copy_(w["d_skip"].reshape(H, Eh))
        m.out_proj.weight.copy_(w["w_out"])
    x, res = synth.activations(2, 20, dims.d_model, seed=5)
    with torch.no_grad():
        hf = m.slow_forward(x).numpy()
    out, _ = M.mixer_forward(dims, _np(w), x.numpy(), res.numpy())
    mine = out - res.numpy()
    assert np.abs(mine - hf).max() / np.abs(hf).max() < 2e-6


def test_zero_weights_and_zero_out_proj_passthrough():
    # SPEC.md:192-193
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, 8, dims.d_model)
    wz = {k: np.zeros_like(v) for k, v in w.items()}
    out, _ = M.mixer_forward(dims, wz, x.numpy(), res.numpy())
    np.testing.assert_array_equal(out, res.numpy())
    w0 = dict(w); w0["w_out"] = np.zeros_like(w["w_out"])
    out, _ = M.mixer_forward(dims, w0, x.numpy(), res.numpy())
    np.testing.assert_array_equal(out, res.numpy())


@pytest.mark.parametrize("L_in,L_out", [(8, 4), (1, 3), (13, 5)])
def test_prefill_then_decode_equals_one_pass(L_in, L_out):
    # PAPER.md:276-280 (§4.1) / SPEC.md:202: prefill(L) + decode(K) == one pass over L+K.
    # The scan and conv are the same fp64 ops in the same order; only BLAS may block the
    # projections differently for different row counts, hence 1e-12 instead of bits.
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, L_in + L_out, dims.d_model, seed=11)
    x, res = x.numpy(), res.numpy()
    full, st_full = M.mixer_forward(dims, w, x, res)
    out, st = M.mixer_prefill(dims, w, x[:, :L_in], res[:, :L_in])
    outs = [out]
    for t in range(L_in, L_in + L_out):
        o, st = M.mixer_decode(dims, w, x[:, t:t + 1], res[:, t:t + 1], st)
        outs.append(o)
    np.testing.assert_allclose(np.concatenate(outs, 1), full, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(st[0], st_full[0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(st[1], st_full[1], rtol=1e-12, atol=1e-12)


def test_chunk_size_invariance():
    # Q19: chunked prefill with the state carried equals one pass
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, 30, dims.d_model, seed=12)
    x, res = x.numpy(), res.numpy()
    full, _ = M.mixer_forward(dims, w, x, res)
    for chunk in (1, 2, 7, 16):
        st, outs = None, []
        for s in range(0, 30, chunk):
            o, st = M.mixer_forward(dims, w, x[:, s:s + chunk], res[:, s:s + chunk], st)
            outs.append(o)
        np.testing.assert_allclose(np.concatenate(outs, 1), full, rtol=1e-12, atol=1e-12)


def test_causality_and_batch_independence():
    # SPEC.md:203, 207
    dims = _tiny()
    w = _np(synth.layer_weights(dims, 0))
    x, res = synth.activations(2, 12, dims.d_model, seed=13)
    x, res = x.numpy(), res.numpy()
    base, _ = M.mixer_forward(dims, w, x, res)
    x2 = x.copy(); x2[:, 7] += 1.0
    pert, _ = M.mixer_forward(dims, w, x2, res)
    np.testing.assert_allclose(pert[:, :7], base[:, :7], rtol=1e-13, atol=1e-13)
    assert np.abs(pert[:, 7:] - base[:, 7:]).max() > 1e-6
    for b in range(2):
        ob, _ = M.mixer_forward(dims, w, x[b:b + 1], res[b:b + 1])
        np.testing.assert_allclose(ob[0], base[b], rtol=1e-13, atol=1e-13)


def test_channel_permutation_equivariance_of_ssm_path():
    # permuting channels of every per-channel input permutes the scan outputs
    rng = np.random.default_rng(9)
    Bsz, L, E, N = 2, 6, 8, 4
    u = rng.standard_normal((Bsz, L, E)); dl = rng.uniform(0.01, 1, (Bsz, L, E))
    A = -np.exp(rng.standard_normal((E, N))); Bm = rng.standard_normal((Bsz, L, N)); Cm = rng.standard_normal((Bsz, L, N))
    Dv = rng.standard_normal(E)
    p = rng.permutation(E)
    y, h = M.scan_full(u, dl, A, Bm, Cm, Dv, np.zeros((Bsz, E, N)))
    yp, hp = M.scan_full(u[:, :, p], dl[:, :, p], A[p], Bm, Cm, Dv[p], np.zeros((Bsz, E, N)))
    np.testing.assert_array_equal(yp, y[:, :, p])
    np.testing.assert_array_equal(hp, h[:, p])


def _hf_block(dims, w, eps):
    """HF MambaBlock (pre-norm RMSNorm -> MambaMixer -> residual add) in float64, norm weight 1."""
    from transformers import MambaConfig
    from transformers.models.mamba.modeling_mamba import MambaBlock
    m = _hf_mamba(dims, w)
    cfg = MambaConfig(hidden_size=dims.d_model, intermediate_size=dims.d_inner, state_size=dims.d_state,
                      conv_kernel=dims.d_conv, time_step_rank=dims.dt_rank, use_bias=False, use_conv_bias=True,
                      hidden_act="silu", use_mambapy=False, layer_norm_epsilon=eps, residual_in_fp32=False)
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    try:
        blk = MambaBlock(cfg, layer_idx=0).eval()
    finally:
        torch.set_default_dtype(prev)
    blk.mixer = m
    with torch.no_grad():
        blk.norm.weight.fill_(1.0)
    return blk


@pytest.mark.parametrize("scale", [1.0, 3e-3])
def test_model_forward_matches_hf_mamba_blocks(scale):
    """oracle.model_forward (the pre-norm stack of reading Q16: residual += mixer(RMSNorm(residual)),
    eps 1e-5, RMSNorm weight 1, residual carried in float64) against two chained HF MambaBlocks in
    float64 (residual_in_fp32=False so no cast).  At scale 3e-3 the residual's mean square (~1e-5)
    is of the order of eps, so a wrong eps, a post-norm order or a residual swap all fail."""
    warnings.filterwarnings("ignore")
    dims = _tiny(n_layers=2)
    ws = [synth.layer_weights(dims, l) for l in range(2)]
    _, res = synth.activations(2, 24, dims.d_model, seed=17)
    res = res * scale
    with torch.no_grad():
        h = res.clone()
        for l in range(2):
            h = _hf_block(dims, ws[l], 1e-5)(h)
    hf = h.numpy()
    mine, _ = M.model_forward(dims, [_np(w) for w in ws], res.numpy(), norm_eps=1e-5)
    d_hf, d_mine = hf - res.numpy(), mine - res.numpy()
    # HF casts A, B, u to fp32 inside the mixer (modeling_mamba.py slow path) -> ~1e-7, not bits
    assert np.abs(d_mine - d_hf).max() / np.abs(d_hf).max() < 2e-6
    # the pins bite: eps 1e-6 (Falcon's mixer eps) instead of 1e-5 is far outside the tolerance
    wrong, _ = M.model_forward(dims, [_np(w) for w in ws], res.numpy(), norm_eps=1e-6)
    assert np.abs((wrong - res.numpy()) - d_hf).max() / np.abs(d_hf).max() > (1e-3 if scale < 1 else 1e-7)
