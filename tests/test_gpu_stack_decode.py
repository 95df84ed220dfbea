"""Persistent whole-stack decode (ssm_stack_decode, csrc/decode_mk.cu) against the fp64 oracle.

One launch runs a decode token through every layer of a pre-norm stack (reading Q16:
residual += mixer(RMSNorm(residual))).  The prompt is prefilled through the per-layer
ssm_mixer_prefill calls (the cache then carries into the persistent decode: PAPER.md:276-287),
and every decode token's residual is compared with oracle.mixer_ref.model_forward over the whole
prompt + decode sequence (tolerance 2e-2 bf16, north_star).  The SSM cache the
kernel leaves behind (h, conv window) is compared with the oracle's final state.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import mixer_ref as M
from paper_2602_21144_b200 import LayerWeights, TPMixer, _lib as L
from paper_2602_21144_b200.stack import MixerStack

from gpu_helpers import TOL, np64, oracle_state_from_gpu_layout, prep_weights, rel

pytestmark = pytest.mark.gpu


def _run(dims, n_layers, B, L_in, L_out, graph=False, seed=5):
    ws = [prep_weights(dims, l, "bf16") for l in range(n_layers)]
    g = torch.Generator().manual_seed(seed)
    res0 = torch.randn(B, L_in + L_out, dims.d_model, generator=g, dtype=torch.float64).float().double()
    mx = TPMixer(dims, "bf16")
    lws = [LayerWeights(dims, w, 1, 0, "bf16").pack(mx) for w in ws]
    st = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8, persistent=True)
    assert st.stack_ws is not None
    pre = res0[:, :L_in].float().cuda().contiguous().view(B * L_in, -1)
    st.prefill_chunk(pre)
    rt = torch.empty(B, dims.d_model, device="cuda")
    launches0 = mx.launches()
    outs = []
    gr = None
    if graph:
        gr = st.capture_decode(rt, warmup=False)
    for t in range(L_in, L_in + L_out):
        rt.copy_(res0[:, t].float().cuda())
        if graph:
            gr.replay()
        else:
            st.decode_step(rt)
        outs.append(rt.cpu().clone())
    st.stack_check()
    if not graph:
        assert mx.launches() - launches0 == L_out  # one kernel per decode token
    ref, ref_states = M.model_forward(dims, [np64(w) for w in ws], res0.numpy())
    r0 = res0.numpy()
    got_dec = torch.stack(outs, 1).double().numpy()
    err = rel(got_dec - r0[:, L_in:], ref[:, L_in:] - r0[:, L_in:])
    assert err < TOL["bf16"], f"decode residual delta rel err {err:.3e}"
    for l in range(n_layers):
        conv, h = oracle_state_from_gpu_layout(st.states[l].conv, st.states[l].h)
        assert rel(h, ref_states[l][1]) < TOL["bf16"], f"layer {l} h"
        assert rel(conv, ref_states[l][0]) < TOL["bf16"], f"layer {l} conv window"
    return err


@pytest.mark.parametrize("B", [1, 7, 16, 24, 32])
def test_stack_decode_small_dims_vs_oracle(B):
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_layers=3)
    _run(dims, 3, B, 10, 4)


def test_stack_decode_falcon_rmsnorm_and_graph_replay():
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_layers=2, bcdt_rmsnorm=True)
    _run(dims, 2, 16, 9, 5, graph=True)


def test_stack_decode_conv_k2_k3():
    for K in (2, 3):
        dims = synth.MixerDims(d_model=128, d_inner=256, dt_rank=16, d_conv=K, n_layers=2)
        _run(dims, 2, 4, 6, 3)


def test_stack_decode_mamba28b_shapes_vs_oracle():
    """Bench shapes (Mamba-2.8B: d_model 2560, d_inner 5120, dt_rank 160) at batch 16 over
    2 layers: every CTA owns in_proj / out_proj units spanning row tiles, ragged channel ranges."""
    dims = synth.MixerDims(d_model=2560, d_inner=5120, dt_rank=160, n_layers=2)
    _run(dims, 2, 16, 3, 2, graph=True)


def test_stack_decode_matches_per_layer_path_over_many_tokens():
    """64 graph-replayed tokens: the persistent kernel and the per-layer decode chain stay
    within bf16 tolerance of each other (no drift of the monotonic barrier / zeroed accumulators)."""
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_layers=4)
    B, L_in, T = 8, 8, 64
    ws = [prep_weights(dims, l, "bf16") for l in range(4)]
    g = torch.Generator().manual_seed(3)
    res0 = torch.randn(B, L_in + T, dims.d_model, generator=g).float()
    mx = TPMixer(dims, "bf16")
    runs = []
    for persistent in (True, False):
        lws = [LayerWeights(dims, w, 1, 0, "bf16").pack(mx) for w in ws]
        st = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8, persistent=persistent)
        assert (st.stack_ws is not None) == persistent
        st.prefill_chunk(res0[:, :L_in].cuda().contiguous().view(B * L_in, -1))
        rt = torch.empty(B, dims.d_model, device="cuda")
        gr = st.capture_decode(rt, warmup=False)
        outs = []
        for t in range(L_in, L_in + T):
            rt.copy_(res0[:, t].cuda())
            gr.replay()
            outs.append(rt.cpu().clone())
        st.stack_check()
        runs.append(torch.stack(outs, 1).double() - res0[:, L_in:].double())
    assert rel(runs[0].numpy(), runs[1].numpy()) < TOL["bf16"]


def test_stack_decode_unsupported_configs_raise():
    mx32 = TPMixer(synth.MixerDims(d_model=256, d_inner=512, dt_rank=16), "fp32")
    import ctypes as C
    nb = C.c_size_t()
    assert L.LIB.ssm_stack_bytes(mx32.handle, 2, 4, C.byref(nb)) == 8  # SSM_ERR_UNSUPPORTED
    mx = TPMixer(synth.MixerDims(d_model=256, d_inner=512, dt_rank=16), "bf16")
    assert L.LIB.ssm_stack_bytes(mx.handle, 2, 33, C.byref(nb)) == 8   # batch > 32
    assert L.LIB.ssm_stack_bytes(mx.handle, 2, 32, C.byref(nb)) == 0
    mxz = TPMixer(synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2), "bf16")
    assert L.LIB.ssm_stack_bytes(mxz.handle, 2, 4, C.byref(nb)) == 8   # two x_proj heads
    # unpacked layers: the stack falls back to per-layer decode unless persistence is required
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16)
    lw = LayerWeights(dims, prep_weights(dims, 0, "bf16"), 1, 0, "bf16")
    assert MixerStack(mx, [lw], 4, 4).stack_ws is None
    assert MixerStack(mx, [lw], 4, 4, persistent=None).stack_ws is None  # opt-in only
    with pytest.raises(L.SSMError):
        MixerStack(mx, [lw], 4, 4, persistent=True)


def test_decode_chain_prenorm_folded_vs_oracle(monkeypatch):
    """Opt-in decode chain (ssm_decode_chain_begin + ssm_mixer_decode_chained): the pre-norm's
    1/rms applied inside the in_proj epilogue and the next layer's bf16 input written by the
    out_proj's last contributor per tile; checked over graph-replayed tokens against the oracle."""
    monkeypatch.setenv("SSM_DECODE_CHAIN", "1")
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_layers=3)
    B, L_in, T = 8, 6, 6
    ws = [prep_weights(dims, l, "bf16") for l in range(3)]
    g = torch.Generator().manual_seed(11)
    res0 = torch.randn(B, L_in + T, dims.d_model, generator=g, dtype=torch.float64).float().double()
    mx = TPMixer(dims, "bf16")
    lws = [LayerWeights(dims, w, 1, 0, "bf16").pack(mx) for w in ws]
    st = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8, persistent=False)
    assert st.chain
    st.prefill_chunk(res0[:, :L_in].float().cuda().contiguous().view(B * L_in, -1))
    rt = torch.empty(B, dims.d_model, device="cuda")
    gr = st.capture_decode(rt, warmup=False)
    outs = []
    for t in range(L_in, L_in + T):
        rt.copy_(res0[:, t].float().cuda())
        gr.replay()
        outs.append(rt.cpu().clone())
    ref, _ = M.model_forward(dims, [np64(w) for w in ws], res0.numpy())
    r0 = res0.numpy()
    got = torch.stack(outs, 1).double().numpy()
    assert rel(got - r0[:, L_in:], ref[:, L_in:] - r0[:, L_in:]) < TOL["bf16"]
