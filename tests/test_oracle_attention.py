"""Pins of oracle/attention_ref.py (Zamba's shared transformer block):
HF transformers ZambaAttentionDecoderLayer (eager attention, float64) + the hybrid layer's linear,
the KV-cache prefix invariant (prefill L + decode K == one pass), causality, and the tensor-parallel
split (heads / MLP columns, two all-reduces) == single rank."""
import warnings

import numpy as np
import pytest
import torch

import synth
from oracle import attention_ref as A

SMALL = synth.AttnDims(d_model=64, n_heads=4, intermediate=96)


def _np(w):
    return {k: v.numpy() for k, v in w.items()}


def _inputs(B, L, D, seed=5):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(B, L, D, generator=g, dtype=torch.float64), torch.randn(B, L, D, generator=g, dtype=torch.float64))


def test_shared_block_matches_hf_zamba_attention_decoder_layer():
    warnings.filterwarnings("ignore")
    from transformers import ZambaConfig
    from transformers.models.zamba.modeling_zamba import ZambaAttentionDecoderLayer
    D, H, I = SMALL.d_model, SMALL.n_heads, SMALL.intermediate
    cfg = ZambaConfig(hidden_size=D, attention_hidden_size=2 * D, num_attention_heads=H, num_key_value_heads=H,
                      attention_head_dim=2 * D // H, intermediate_size=I, hidden_act="gelu", rms_norm_eps=1e-5)
    cfg._attn_implementation = "eager"
    w = synth.shared_block_weights(SMALL)
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    try:
        layer = ZambaAttentionDecoderLayer(cfg, layer_idx=0).eval()
    finally:
        torch.set_default_dtype(prev)
    with torch.no_grad():
        layer.input_layernorm.weight.copy_(w["norm1"])
        layer.self_attn.q_proj.weight.copy_(w["w_q"])
        layer.self_attn.k_proj.weight.copy_(w["w_k"])
        layer.self_attn.v_proj.weight.copy_(w["w_v"])
        layer.self_attn.o_proj.weight.copy_(w["w_o"])
        layer.pre_ff_layernorm.weight.copy_(w["norm2"])
        layer.feed_forward.gate_proj.weight.copy_(w["w_g"])
        layer.feed_forward.up_proj.weight.copy_(w["w_u"])
        layer.feed_forward.down_proj.weight.copy_(w["w_d"])
    B, L = 2, 12
    h, h0 = _inputs(B, L, D)
    mask = torch.full((L, L), float("-inf"), dtype=torch.float64).triu(1)[None, None].expand(B, 1, L, L)
    with torch.no_grad():
        hf = layer(h, original_hidden_states=h0, layer_idx=0, attention_mask=mask) @ w["w_lin"].T
    mine, _ = A.shared_block(SMALL, _np(w), h.numpy(), h0.numpy())
    # HF casts to float32 inside ZambaRMSNorm and the softmax (modeling_zamba.py) -> ~1e-7, not bits
    assert np.abs(mine - hf.numpy()).max() / np.abs(hf.numpy()).max() < 1e-6


def test_kv_cache_prefill_then_decode_equals_one_pass():
    w = _np(synth.shared_block_weights(SMALL))
    h, h0 = _inputs(2, 10, SMALL.d_model, seed=6)
    full, kv_full = A.shared_block(SMALL, w, h.numpy(), h0.numpy())
    out, kv = A.shared_block(SMALL, w, h[:, :6].numpy(), h0[:, :6].numpy())
    outs = [out]
    for t in range(6, 10):
        o, kv = A.shared_block(SMALL, w, h[:, t:t + 1].numpy(), h0[:, t:t + 1].numpy(), kv)
        outs.append(o)
    np.testing.assert_allclose(np.concatenate(outs, 1), full, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(kv[0], kv_full[0], rtol=1e-12, atol=1e-12)


def test_causality():
    w = _np(synth.shared_block_weights(SMALL))
    h, h0 = _inputs(1, 8, SMALL.d_model, seed=7)
    a, _ = A.shared_block(SMALL, w, h.numpy(), h0.numpy())
    h2 = h.clone()
    h2[:, 5:] += 1.0
    b, _ = A.shared_block(SMALL, w, h2.numpy(), h0.numpy())
    np.testing.assert_array_equal(a[:, :5], b[:, :5])
    assert np.abs(a[:, 5:] - b[:, 5:]).max() > 1e-3


@pytest.mark.parametrize("k", [2, 4])
def test_tensor_parallel_split_equals_single_rank(k):
    w = _np(synth.shared_block_weights(SMALL))
    h, h0 = _inputs(2, 7, SMALL.d_model, seed=8)
    ref, kv = A.shared_block(SMALL, w, h.numpy(), h0.numpy())
    tp, shards = A.shared_block_tp(SMALL, w, h.numpy(), h0.numpy(), k)
    np.testing.assert_allclose(tp, ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.concatenate([s[0] for s in shards], 2), kv[0], rtol=1e-12, atol=1e-12)


def test_gelu_closed_forms():
    g = A.gelu(np.array([0.0, 1.0, -1.0]))
    assert g[0] == 0.0
    np.testing.assert_allclose(g[1], 0.8413447460685429, rtol=1e-15)       # Phi(1)
    np.testing.assert_allclose(g[2], -0.15865525393145707, rtol=1e-15)    # -(1 - Phi(1))
