"""Oracle parity of the persistent whole-stack decode (ssm_dstack_*).

One cooperative launch per token runs every layer's pre-norm decode block from the caches that the
chunked prefill filled; the result must equal the fp64 pre-norm stack oracle (oracle.model_forward,
pinned to HF MambaBlock in tests/test_oracle_mixer.py) over prompt + generated tokens in one pass
(the prefix/cache invariant), at 2e-2 (bf16 I/O, fp32 state).  Covered: several grid sizes (every SM,
odd CTA counts that leave CTAs without units / channels), ragged batches (1, 7, 16), d_conv 2..4,
Falcon-Mamba's dt/B/C RMSNorm (reading Q18), CUDA-graph replay, the bench's Mamba-2.8B shape, and
agreement with the per-layer decode path.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import mixer_ref as M
from paper_2602_21144_b200 import LayerWeights, SSMError, TPMixer, _lib as L
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer
from gpu_helpers import TOL, rel

pytestmark = pytest.mark.gpu


def _host_weights(full):
    out = {}
    for k, v in full.items():
        v = v.detach().cpu().to(torch.float64)
        out[k] = synth.bf16_round(v).numpy() if k in ("w_in", "w_x", "w_dt", "w_out") else \
            v.to(torch.float32).to(torch.float64).numpy()
    return out


def _run(dims, B, L_in, L_out, ctas=0, graph=False, seed=3):
    mx = TPMixer(dims, "bf16")
    fulls = [synthetic_layer(dims, l, seed=1000 + seed) for l in range(dims.n_layers)]
    lws = [LayerWeights(dims, f, 1, 0, "bf16") for f in fulls]
    ws = [_host_weights(f) for f in fulls]
    del fulls
    stack = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8).persistent(ctas)
    g = torch.Generator().manual_seed(seed)
    res0 = torch.randn(B, L_in + L_out, dims.d_model, generator=g, dtype=torch.float64).float()
    pre = res0[:, :L_in].cuda().contiguous().view(B * L_in, -1)
    res_t = torch.empty(B, dims.d_model, device="cuda")
    gr = None
    if graph:
        res_t.copy_(res0[:, L_in].cuda())
        gr = stack.capture_decode(res_t)        # (its warm-up step advances the caches: prefill again)
        assert stack.graph_launches == 1
        stack.reset()
    stack.prefill_chunk(pre)
    outs = []
    for t in range(L_in, L_in + L_out):
        res_t.copy_(res0[:, t].cuda())
        if gr is not None:
            stack.replay(gr)
        else:
            stack.decode_step(res_t)
        outs.append(res_t.cpu().clone())
    torch.cuda.synchronize()
    got_pre = pre.view(B, L_in, -1).cpu().double().numpy()
    got_dec = torch.stack(outs, 1).double().numpy()
    r0 = res0.double().numpy()
    ref, _ = M.model_forward(dims, ws, r0)
    assert rel(got_pre - r0[:, :L_in], ref[:, :L_in] - r0[:, :L_in]) < TOL["bf16"]
    err = rel(got_dec - r0[:, L_in:], ref[:, L_in:] - r0[:, L_in:])
    assert err < TOL["bf16"], err
    return stack, got_dec, err


SMALL = dict(d_model=256, d_inner=512, dt_rank=16, n_layers=3)


@pytest.mark.parametrize("ctas", [0, 15, 37, 129])
def test_dstack_small_vs_model_forward_grid_sizes(ctas):
    _run(synth.MixerDims(**SMALL), B=4, L_in=24, L_out=6, ctas=ctas)


@pytest.mark.parametrize("B", [1, 7, 16])
def test_dstack_ragged_batch(B):
    _run(synth.MixerDims(**SMALL), B=B, L_in=16, L_out=5)


@pytest.mark.parametrize("K", [2, 3])
def test_dstack_conv_widths(K):
    _run(synth.MixerDims(**{**SMALL, "d_conv": K}), B=3, L_in=9, L_out=5)


def test_dstack_falcon_bcdt_rmsnorm():
    _run(synth.MixerDims(**{**SMALL, "dt_rank": 32, "bcdt_rmsnorm": True}), B=5, L_in=12, L_out=5)


def test_dstack_graph_replay():
    _run(synth.MixerDims(**SMALL), B=4, L_in=20, L_out=6, graph=True)


def test_dstack_mamba28b_two_layers_bench_path():
    """The bench's shape and launch configuration: Mamba-2.8B dims (D 2560, E 5120, R 160), batch 16,
    every SM, graph replay."""
    dims = synth.MixerDims(**{**synth.CONFIGS["mamba2.8b"].asdict(), "n_layers": 2})
    _run(dims, B=16, L_in=32, L_out=5, graph=True)


def test_dstack_agrees_with_per_layer_decode():
    """Same caches and inputs through the per-layer graph path and the persistent kernel: the two
    CUDA paths agree far inside the oracle tolerance."""
    dims = synth.MixerDims(**SMALL)
    B, L_in, L_out = 4, 16, 4
    mx = TPMixer(dims, "bf16")
    fulls = [synthetic_layer(dims, l) for l in range(dims.n_layers)]
    lws = [LayerWeights(dims, f, 1, 0, "bf16") for f in fulls]
    g = torch.Generator().manual_seed(11)
    res0 = torch.randn(B, L_in + L_out, dims.d_model, generator=g).cuda()
    outs = []
    for persistent in (False, True):
        st = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8)
        if persistent:
            st.persistent()
        pre = res0[:, :L_in].contiguous().view(B * L_in, -1)
        st.prefill_chunk(pre)
        r = torch.empty(B, dims.d_model, device="cuda")
        o = []
        for t in range(L_in, L_in + L_out):
            r.copy_(res0[:, t])
            st.decode_step(r)
            o.append(r.clone())
        outs.append(torch.stack(o, 1) - res0[:, L_in:])
    torch.cuda.synchronize()
    assert rel(outs[1].cpu().numpy(), outs[0].cpu().numpy()) < 5e-3


def test_dstack_unsupported_shapes_raise():
    mx = TPMixer(synth.MixerDims(**SMALL), "bf16")
    lws = [LayerWeights(synth.MixerDims(**SMALL), synthetic_layer(synth.MixerDims(**SMALL), 0), 1, 0, "bf16")]
    with pytest.raises(SSMError):
        MixerStack(mx, lws, 17, 4, L.SSM_AR2_INT8).persistent()            # batch > 16
    with pytest.raises(SSMError):
        MixerStack(mx, lws, 2, 4, L.SSM_AR2_INT8).persistent(ctas=100000)  # more CTAs than SMs
    mxf = TPMixer(synth.MixerDims(**SMALL), "fp32")
    lwf = [LayerWeights(synth.MixerDims(**SMALL), synthetic_layer(synth.MixerDims(**SMALL), 0), 1, 0, "fp32")]
    with pytest.raises(SSMError):
        MixerStack(mxf, lwf, 2, 4, L.SSM_AR2_INT8).persistent()            # fp32 mode
    zd = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2)
    mxz = TPMixer(zd, "bf16")
    lwz = [LayerWeights(zd, synthetic_layer(zd, 0), 1, 0, "bf16")]
    with pytest.raises(SSMError):
        MixerStack(mxz, lwz, 2, 4, L.SSM_AR2_INT8).persistent()            # two x_proj heads (Zamba)
    np.testing.assert_(True)
