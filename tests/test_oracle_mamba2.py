"""Pins of oracle/mamba2_ref.py (Mamba-2 SSD mixer):
HF transformers Mamba2Mixer.torch_forward in float64 (its chunked State-Space-Duality matrix form,
an independent formulation of the recurrence the oracle writes per timestep), the prefix/cache
invariant, and the tensor-parallel split (heads; replicated B/C; all-reduced norm statistics and
out_proj partials) == single rank."""
import warnings

import numpy as np
import pytest
import torch

import synth
from oracle import mamba2_ref as M2

SMALL = synth.Mamba2Dims(d_model=64, d_inner=128, d_state=16, headdim=16, n_groups=1)


def _np(w):
    return {k: v.numpy() for k, v in w.items()}


@pytest.mark.parametrize("L,chunk", [(24, 8), (21, 16)])
def test_matches_hf_mamba2_torch_forward(L, chunk):
    warnings.filterwarnings("ignore")
    from transformers import Mamba2Config
    from transformers.models.mamba2.modeling_mamba2 import Mamba2Mixer
    m2 = SMALL
    cfg = Mamba2Config(hidden_size=m2.d_model, num_heads=m2.n_heads, head_dim=m2.headdim, expand=2,
                       state_size=m2.d_state, n_groups=m2.n_groups, conv_kernel=m2.d_conv, chunk_size=chunk,
                       use_bias=False, use_conv_bias=True, layer_norm_epsilon=m2.eps, hidden_act="silu")
    w = synth.mamba2_weights(m2)
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    try:
        mix = Mamba2Mixer(cfg, layer_idx=0).eval()
    finally:
        torch.set_default_dtype(prev)
    with torch.no_grad():
        mix.in_proj.weight.copy_(w["w_in"])
        mix.conv1d.weight.copy_(w["conv_w"][:, None, :])
        mix.conv1d.bias.copy_(w["conv_b"])
        mix.dt_bias.copy_(w["dt_bias"])
        mix.A_log.copy_(w["a_log"])
        mix.D.copy_(w["d_skip"])
        mix.norm.weight.copy_(w["norm_w"])
        mix.out_proj.weight.copy_(w["w_out"])
    x, res = synth.activations(2, L, m2.d_model, seed=4)
    with torch.no_grad():
        hf = mix.torch_forward(x).numpy()
    out, _ = M2.mixer_forward(m2, _np(w), x.numpy(), res.numpy())
    mine = out - res.numpy()
    # HF's gated RMSNorm computes in float32 (MambaRMSNormGated) -> ~1e-7, not bits
    assert np.abs(mine - hf).max() / np.abs(hf).max() < 1e-6


def test_prefill_then_decode_equals_one_pass():
    w = _np(synth.mamba2_weights(SMALL))
    x, res = synth.activations(2, 14, SMALL.d_model, seed=5)
    full, st_full = M2.mixer_forward(SMALL, w, x.numpy(), res.numpy())
    out, st = M2.mixer_forward(SMALL, w, x[:, :9].numpy(), res[:, :9].numpy())
    outs = [out]
    for t in range(9, 14):
        o, st = M2.mixer_forward(SMALL, w, x[:, t:t + 1].numpy(), res[:, t:t + 1].numpy(), st)
        outs.append(o)
    np.testing.assert_allclose(np.concatenate(outs, 1), full, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(st[1], st_full[1], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("k", [2, 4])
def test_tensor_parallel_equals_single_rank(k):
    w = _np(synth.mamba2_weights(SMALL))
    x, res = synth.activations(2, 10, SMALL.d_model, seed=6)
    ref, _ = M2.mixer_forward(SMALL, w, x.numpy(), res.numpy())
    tp = M2.mixer_forward_tp(SMALL, w, x.numpy(), res.numpy(), k)
    np.testing.assert_allclose(tp, ref, rtol=1e-12, atol=1e-12)


def test_zero_input_decays_state():
    """With u = 0 the state only decays: |h_t| = exp(sum dt A) |h_0| < |h_0| (A < 0, dt > 0)."""
    w = _np(synth.mamba2_weights(SMALL))
    w["w_in"] = np.zeros_like(w["w_in"])          # x = B = C = dt_raw = 0 before the conv bias
    w["conv_b"] = np.full_like(w["conv_b"], -40.0)  # SiLU(-40) ~ 0: x, B, C ~ 0
    H, P, N = SMALL.n_heads, SMALL.headdim, SMALL.d_state
    h0 = np.random.default_rng(0).standard_normal((1, H, P, N))
    st = (np.zeros((1, SMALL.d_inner + 2 * N, SMALL.d_conv - 1)), h0)
    x, res = synth.activations(1, 3, SMALL.d_model, seed=7)
    _, (_, h) = M2.mixer_forward(SMALL, w, x.numpy(), res.numpy(), st)
    assert np.all(np.abs(h) <= np.abs(h0) + 1e-12) and np.abs(h).max() < np.abs(h0).max()
