"""GPU parity of Zamba's shared transformer block through
ssm_attn_block: chunked prefill then token-by-token decode from the KV cache, at TP = 1 and on
virtual TP = 2 / 4 ranks (heads and MLP columns split, two all-reduces), against the fp64 oracle
(oracle/attention_ref.py, pinned to HF ZambaAttentionDecoderLayer), tolerance 2e-2 (bf16 I/O)."""
import numpy as np
import pytest
import torch

import synth
from oracle import attention_ref as A
from paper_2602_21144_b200 import TPMixer, _lib as L
from paper_2602_21144_b200.attention import SharedBlock, SharedBlockWeights
from gpu_helpers import TOL, VirtualGroup, rel

pytestmark = pytest.mark.gpu


def _host(w):
    mats = ("w_q", "w_k", "w_v", "w_o", "w_g", "w_u", "w_d", "w_lin")
    return {k: (synth.bf16_round(v) if k in mats else v.float().double()).numpy() for k, v in w.items()}


def _run(adims, k, B, chunks, n_dec, flags=0, seed=11):
    D = adims.d_model
    T = sum(chunks) + n_dec
    w = synth.shared_block_weights(adims)
    g = torch.Generator().manual_seed(seed)
    h = torch.randn(B, T, D, generator=g, dtype=torch.float64).float()
    h0 = torch.randn(B, T, D, generator=g, dtype=torch.float64).float()
    mdims = synth.MixerDims(d_model=D, d_inner=2 * D, dt_rank=max(16, D // 16))
    if k == 1:
        grp = None
        mixers = [TPMixer(mdims, "bf16")]
    else:
        grp = VirtualGroup(mdims, k, "bf16", B * max(chunks))
        mixers = grp.mixers
    ws = [SharedBlockWeights(adims, w, k, r) for r in range(k)]
    blocks = [SharedBlock(mixers[r], adims, B, T, max(chunks)) for r in range(k)]
    steps = [(t0, c) for t0, c in zip(np.cumsum([0] + chunks[:-1]), chunks)] + \
            [(sum(chunks) + j, 1) for j in range(n_dec)]
    outs = [[] for _ in range(k)]
    for t0, c in steps:
        hs = [h[:, t0:t0 + c].cuda().contiguous().view(B * c, D) for _ in range(k)]
        h0s = [h0[:, t0:t0 + c].cuda().contiguous().view(B * c, D) for _ in range(k)]
        ts = [torch.empty(B * c, D, device="cuda") for _ in range(k)]
        torch.cuda.synchronize()
        if grp is None:
            blocks[0](ws[0], hs[0], h0s[0], ts[0], c, flags)
            torch.cuda.synchronize()
        else:
            grp.run(lambda r, mx, s: blocks[r](ws[r], hs[r], h0s[r], ts[r], c, flags, s))
        for r in range(k):
            outs[r].append(ts[r].view(B, c, D).cpu())
    got = [torch.cat(o, 1).double().numpy() for o in outs]
    ref, _ = A.shared_block(adims, _host(w), h.double().numpy(), h0.double().numpy())
    return got, ref


@pytest.mark.parametrize("D,H,I", [(64, 4, 96), (128, 4, 192), (256, 4, 256)])
def test_shared_block_tp1_prefill_decode_vs_oracle(D, H, I):
    adims = synth.AttnDims(d_model=D, n_heads=H, intermediate=I)
    got, ref = _run(adims, 1, 2, [40, 29], 4)
    assert rel(got[0], ref) < TOL["bf16"]


def test_shared_block_zamba7b_head_dim_464():
    """The Zamba-7B shape (D 3712, 16 heads of 464, MLP 14848): 70 query rows span two 64-row
    tiles and two key tiles (causal), then decode tokens."""
    got, ref = _run(synth.ZAMBA7B_ATTN, 1, 1, [70], 3)
    assert rel(got[0], ref) < TOL["bf16"]


@pytest.mark.parametrize("k,flags", [(2, 0), (4, 0), (2, L.SSM_AR2_INT8)])
def test_shared_block_virtual_tp_vs_oracle(k, flags):
    adims = synth.AttnDims(d_model=128, n_heads=8, intermediate=256)
    got, ref = _run(adims, k, 2, [33, 31], 3, flags)
    for r in range(1, k):
        np.testing.assert_array_equal(got[r], got[0])      # replicas bitwise identical
    assert rel(got[0], ref) < TOL["bf16"]


def test_kv_overflow_reports_and_reset_empties():
    adims = synth.AttnDims(d_model=64, n_heads=4, intermediate=96)
    mx = TPMixer(synth.MixerDims(d_model=64, d_inner=128, dt_rank=4), "bf16")
    blk = SharedBlock(mx, adims, 1, 8, 8)
    w = SharedBlockWeights(adims, synth.shared_block_weights(adims))
    x = torch.randn(8, 64, device="cuda")
    t = torch.empty(8, 64, device="cuda")
    blk(w, x, x, t, 8)
    blk(w, x[:1], x[:1], t[:1], 1)     # 9th token: overflow -> error word set
    torch.cuda.synchronize()
    assert int(blk.kv_buf[4:8].view(torch.int32).cpu()[0]) == 1
    blk.reset()
    blk(w, x, x, t, 8)
    torch.cuda.synchronize()
    assert int(blk.kv_buf[0:4].view(torch.int32).cpu()[0]) == 8


@pytest.mark.parametrize("k", [1, 2])
def test_zamba_hybrid_stack_prefill_graph_decode_vs_oracle(k):
    """A Zamba-shaped stack (2 mixer heads; layer 1 of 3 is hybrid: the shared block runs on
    (residual, h0) into t and the Mamba layer takes RMSNorm(residual + t)) through MixerStack: chunked
    prefill, then CUDA-graph decode replays, against the fp64 composition of the oracles."""
    from oracle import mixer_ref as M
    from paper_2602_21144_b200 import LayerWeights
    from paper_2602_21144_b200.attention import hybrid_config
    from paper_2602_21144_b200.stack import MixerStack, synthetic_layer
    from test_gpu_paths import _host_weights
    dims = synth.MixerDims(d_model=128, d_inner=256, dt_rank=16, n_heads=2, n_layers=3)
    adims = synth.AttnDims(d_model=128, n_heads=4, intermediate=256)
    B, L_in, L_out, hyb = 2, 20, 3, 1
    fulls = [synthetic_layer(dims, l) for l in range(3)]
    blk = synth.shared_block_weights(adims)
    lin = {hyb: blk["w_lin"]}
    g = torch.Generator().manual_seed(3)
    res0 = torch.randn(B, L_in + L_out, 128, generator=g, dtype=torch.float64).float()
    h0 = torch.randn(B, L_in + L_out, 128, generator=g, dtype=torch.float64).float()
    grp = VirtualGroup(dims, k, "bf16", B * L_in) if k > 1 else None
    mixers = grp.mixers if k > 1 else [TPMixer(dims, "bf16")]
    stacks = [MixerStack(mixers[r], [LayerWeights(dims, f, k, r, "bf16") for f in fulls], B, L_in, L.SSM_AR2_FP32,
                         hybrid=hybrid_config(adims, blk, lin, k, r, L_in + L_out + 4)) for r in range(k)]
    pre = [res0[:, :L_in].cuda().contiguous().view(B * L_in, -1) for _ in range(k)]
    h0p = [h0[:, :L_in].cuda().contiguous().view(B * L_in, -1) for _ in range(k)]
    rts = [torch.empty(B, 128, device="cuda") for _ in range(k)]
    torch.cuda.synchronize()

    def run(fn):
        if grp is None:
            fn(0, mixers[0], torch.cuda.current_stream())
            torch.cuda.synchronize()
        else:
            grp.run(fn)
    graphs = []
    for r in range(k):
        if grp is None:
            graphs.append(stacks[r].capture_decode(rts[r]))
        else:
            with torch.cuda.stream(grp.streams[r]):
                graphs.append(stacks[r].capture_decode(rts[r], warmup=False))
    run(lambda r, mx, s: (stacks[r].reset(s), stacks[r].prefill_chunk(pre[r], s, h0=h0p[r])))
    outs = []
    for t in range(L_in, L_in + L_out):
        for r in range(k):
            rts[r].copy_(res0[:, t].cuda())
            stacks[r].h0_dec.copy_(h0[:, t].cuda())
        torch.cuda.synchronize()
        run(lambda r, mx, s: stacks[r].replay(graphs[r], s))
        outs.append(rts[0].cpu().clone())
    ws = [_host_weights(f) for f in fulls]
    hb = {kk: (synth.bf16_round(v) if kk.startswith("w_") else v.float().double()).numpy() for kk, v in blk.items()}
    res = res0.double().numpy()
    for l in range(3):
        if l == hyb:
            tt, _ = A.shared_block(adims, hb, res, h0.double().numpy())
            x = M.rmsnorm(res + tt, None, 1e-5)
        else:
            x = M.rmsnorm(res, None, 1e-5)
        res, _ = M.mixer_forward(dims, ws[l], x, res)
    r0 = res0.double().numpy()
    got_pre = pre[0].view(B, L_in, -1).cpu().double().numpy()
    got_dec = torch.stack(outs, 1).double().numpy()
    assert rel(got_pre - r0[:, :L_in], res[:, :L_in] - r0[:, :L_in]) < TOL["bf16"]
    assert rel(got_dec - r0[:, L_in:], res[:, L_in:] - r0[:, L_in:]) < TOL["bf16"]
