"""Oracle parity of the exact configurations the bench and the harness run (round-2 additions):

* the bench's decode path at Mamba-2.8B dimensions: MixerStack over pre-tiled (packed) weights,
  chunk-major prefill, then CUDA-graph replays of the per-layer decode step (fused in_proj with
  the conv step and x_proj in its epilogue, XPN = 3, PDL on at TP = 1) against the fp64 pre-norm
  stack oracle.model_forward (pinned to HF MambaBlock, tests/test_oracle_mixer.py);
* Falcon-Mamba's dt/B/C RMSNorm (reading Q18) at virtual TP = 2 / 4 (applied after AR#1);
* the generation harness's logits (embedding -> stack -> final RMSNorm -> LM head) against an
  fp64 oracle forward of the same sequence (PAPER.md:591-610 structure).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import mixer_ref as M
from paper_2602_21144_b200 import LayerWeights, TPMixer, _lib as L
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer
from gpu_helpers import TOL, np64, rel
from test_gpu_parity import _tp_virtual

pytestmark = pytest.mark.gpu


def _host_weights(full):
    """Device fp32 synthetic weights -> the float64 values the kernels see (matrices bf16)."""
    out = {}
    for k, v in full.items():
        v = v.detach().cpu().to(torch.float64)
        out[k] = synth.bf16_round(v).numpy() if k in ("w_in", "w_x", "w_dt", "w_out") else \
            v.to(torch.float32).to(torch.float64).numpy()
    return out


def test_bench_decode_path_mamba28b_two_layers_vs_model_forward():
    dims = synth.MixerDims(**{**synth.CONFIGS["mamba2.8b"].asdict(), "n_layers": 2})
    B, L_in, L_out = synth.WORKLOADS["mamba2.8b"]["batch"], 64, 5
    mx = TPMixer(dims, "bf16")
    fulls = [synthetic_layer(dims, l) for l in range(2)]
    lws = [LayerWeights(dims, f, 1, 0, "bf16").pack(mx) for f in fulls]    # as bench.py
    ws = [_host_weights(f) for f in fulls]
    del fulls
    stack = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8)
    g = torch.Generator().manual_seed(8)
    res0 = torch.randn(B, L_in + L_out, dims.d_model, generator=g, dtype=torch.float64).float()
    pre = res0[:, :L_in].cuda().contiguous().view(B * L_in, -1)
    stack.prefill_chunk(pre)
    res_t = torch.empty(B, dims.d_model, device="cuda")
    res_t.copy_(res0[:, L_in].cuda())
    probe_graph = stack.capture_decode(res_t, probes=[("in_proj_decode", 2)])   # as bench.py
    graph = stack.capture_decode(res_t, warmup=False)
    assert stack.graph_launches == 2 * 4          # per layer: norm, fused in_proj, decode step, out_proj
    del probe_graph
    # capture_decode's warm-up step advanced the cache by one token: redo the prefill from zero
    stack.reset()
    pre.copy_(res0[:, :L_in].cuda().view(B * L_in, -1))
    stack.prefill_chunk(pre)
    outs = []
    for t in range(L_in, L_in + L_out):
        res_t.copy_(res0[:, t].cuda())
        stack.replay(graph)
        outs.append(res_t.cpu().clone())
    torch.cuda.synchronize()
    assert mx.fused_calls() > 0
    got_pre = pre.view(B, L_in, -1).cpu().double().numpy()
    got_dec = torch.stack(outs, 1).double().numpy()
    r0 = res0.double().numpy()
    for b in (0, B - 1):                        # rows are independent
        ref, _ = M.model_forward(dims, ws, r0[b:b + 1])
        assert rel(got_pre[b] - r0[b, :L_in], ref[0, :L_in] - r0[b, :L_in]) < TOL["bf16"], b
        assert rel(got_dec[b] - r0[b, L_in:], ref[0, L_in:] - r0[b, L_in:]) < TOL["bf16"], b


@pytest.mark.parametrize("k,mode", [(2, "int8"), (4, "int8"), (4, "fp32")])
def test_virtual_tp_falcon_bcdt_rmsnorm_vs_oracle(k, mode):
    """Falcon-Mamba's weightless dt/B/C RMSNorm (eps 1e-6) runs after AR#1 on the summed dbc, in
    the prefill unpack kernel and in the decode step (reading Q18)."""
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, bcdt_rmsnorm=True)
    flags = L.SSM_AR2_INT8 if mode == "int8" else L.SSM_AR2_FP32
    outs, w, x, res, grp, sts = _tp_virtual(dims, "bf16", k, 2, 40, 4, flags)
    for r in range(1, k):
        assert torch.equal(outs[r], outs[0])
    ref, st_ref = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    assert rel(outs[0].double().numpy() - resn, ref - resn) < TOL["bf16"]
    h = np.concatenate([sts[r].h.cpu().double().numpy() for r in range(k)], 1)
    assert rel(h, st_ref[1]) < TOL["bf16"]


@pytest.mark.parametrize("k,arm", [(1, "fp32"), (2, "fp32"), (2, "int8")])
def test_generation_harness_logits_vs_oracle(k, arm):
    """TPLanguageModel logits (teacher-forced) == fp64 oracle: embedding rows as the residual
    stream -> model_forward over prompt + fed tokens (the cache carries prefill into decode, so
    decode positions equal one pass) -> final RMSNorm (eps 1e-5, weight 1) -> LM head."""
    from paper_2602_21144_b200.generate import TPLanguageModel
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_layers=2)
    vocab, B, Lp, n_out = 300, 2, 20, 5
    fulls = [synthetic_layer(dims, l) for l in range(2)]
    g = torch.Generator(device="cuda").manual_seed(4)
    emb = torch.randn(vocab, dims.d_model, generator=g, device="cuda").to(torch.bfloat16)
    head = (torch.randn(vocab, dims.d_model, generator=g, device="cuda") / 16).to(torch.bfloat16)
    prompt = torch.randint(0, vocab, (B, Lp), generator=g, device="cuda")
    forced = torch.randint(0, vocab, (B, n_out), generator=g, device="cuda")
    flags = {"fp32": L.SSM_AR2_FP32, "int8": L.SSM_AR2_INT8}[arm]
    m = TPLanguageModel(dims, fulls, emb, k, flags, B, Lp, head=head)
    _, logits = m.generate(prompt, n_out, forced=forced)      # [n_out, B, vocab]
    seq = torch.cat([prompt, forced[:, :n_out - 1]], 1).cpu()
    e64 = emb.cpu().double().numpy()
    res0 = e64[seq.numpy()]                                   # [B, Lp + n_out - 1, D]
    ref, _ = M.model_forward(dims, [_host_weights(f) for f in fulls], res0)
    xf = M.rmsnorm(ref[:, Lp - 1:], None, 1e-5)
    want = xf @ head.cpu().double().numpy().T                 # [B, n_out, vocab]
    got = logits.permute(1, 0, 2).double().numpy()
    assert rel(got, want) < TOL["bf16"]
    # the oracle's top-1 matches the harness's at (nearly) every position
    agree = (got.argmax(-1) == want.argmax(-1)).mean()
    assert agree >= 0.9


@pytest.mark.parametrize("dims_name,B", [("med", 1), ("med", 16), ("med", 17), ("med", 32), ("med_falcon", 8),
                                         ("med_zamba", 16), ("med_zamba_wide", 4)])
def test_decode_block_variants_vs_oracle(dims_name, B):
    """ssm_mixer_decode_block through MixerStack (eager steps): the default path (fused in_proj for
    batch <= 32) and SSM_DECODE_UNFUSED (plain kernel chain) match the fp64 pre-norm stack and each
    other."""
    dims = {"med": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_layers=2),
            "med_falcon": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, bcdt_rmsnorm=True, n_layers=2),
            "med_zamba": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2, n_layers=2),
            "med_zamba_wide": synth.MixerDims(d_model=256, d_inner=512, dt_rank=232, n_heads=2, n_layers=2)}[dims_name]
    L_in, L_out = 10, 4
    fulls = [synthetic_layer(dims, l) for l in range(2)]
    ws = [_host_weights(f) for f in fulls]
    g = torch.Generator().manual_seed(31)
    res0 = torch.randn(B, L_in + L_out, dims.d_model, generator=g, dtype=torch.float64).float()
    r0 = res0.double().numpy()
    ref, _ = M.model_forward(dims, ws, r0)
    got = {}
    for name, fl in (("default", 0), ("unfused", L.SSM_DECODE_UNFUSED)):
        mx = TPMixer(dims, "bf16")
        lws = [LayerWeights(dims, f, 1, 0, "bf16").pack(mx) for f in fulls]
        stack = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8)
        stack.dec_flags = fl
        pre = res0[:, :L_in].cuda().contiguous().view(B * L_in, -1)
        stack.prefill_chunk(pre)
        outs = []
        rt = torch.empty(B, dims.d_model, device="cuda")
        for t in range(L_in, L_in + L_out):
            rt.copy_(res0[:, t].cuda())
            stack.decode_step(rt)
            outs.append(rt.cpu().clone())
        torch.cuda.synchronize()
        dec = torch.stack(outs, 1).double().numpy()
        assert rel(dec - r0[:, L_in:], ref[:, L_in:] - r0[:, L_in:]) < TOL["bf16"], name
        assert (mx.fused_calls() > 0) == (name != "unfused" and B <= 32)
        got[name] = dec
    d_ref = got["unfused"] - r0[:, L_in:]
    for name in ("default",):
        assert rel(got[name] - r0[:, L_in:], d_ref) < (1e-2 if dims.bcdt_rmsnorm else 5e-3), name


def test_bench_prefill_path_cta_pairs_normed_persistent_vs_model_forward():
    """The bench's exact TP = 1 path at Mamba-2.8B dimensions with a prefill big enough for the
    default CTA-pair GEMMs (batch 16 x 256 = 4096 rows): pre-norm folded around the projections
    (rowstats, in_proj row scale, out_proj epilogue writing the next layer's bf16 input and sums of
    squares), x_proj epilogue splitting dt_low / B || C (no unpack), TMA conv and scan tiles; then
    the persistent whole-stack decode.  Sampled batch rows vs the fp64 oracle stack."""
    dims = synth.MixerDims(**{**synth.CONFIGS["mamba2.8b"].asdict(), "n_layers": 2})
    B, L_in, L_out = synth.WORKLOADS["mamba2.8b"]["batch"], 256, 3
    mx = TPMixer(dims, "bf16")
    fulls = [synthetic_layer(dims, l) for l in range(2)]
    lws = [LayerWeights(dims, f, 1, 0, "bf16") for f in fulls]
    ws = [_host_weights(f) for f in fulls]
    del fulls
    stack = MixerStack(mx, lws, B, L_in, L.SSM_AR2_INT8)
    assert stack.prefill_normed
    stack.persistent()
    g = torch.Generator().manual_seed(9)
    res0 = torch.randn(B, L_in + L_out, dims.d_model, generator=g, dtype=torch.float64).float()
    pre = res0[:, :L_in].cuda().contiguous().view(B * L_in, -1)
    stack.prefill_chunk(pre)
    outs = []
    res_t = torch.empty(B, dims.d_model, device="cuda")
    for t in range(L_in, L_in + L_out):
        res_t.copy_(res0[:, t].cuda())
        stack.decode_step(res_t)
        outs.append(res_t.cpu().clone())
    torch.cuda.synchronize()
    got_pre = pre.view(B, L_in, -1).cpu().double().numpy()
    got_dec = torch.stack(outs, 1).double().numpy()
    r0 = res0.double().numpy()
    for b in (0, B - 1):
        ref, _ = M.model_forward(dims, ws, r0[b:b + 1])
        assert rel(got_pre[b] - r0[b, :L_in], ref[0, :L_in] - r0[b, :L_in]) < TOL["bf16"], b
        assert rel(got_dec[b] - r0[b, L_in:], ref[0, L_in:] - r0[b, L_in:]) < TOL["bf16"], b
