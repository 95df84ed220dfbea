"""Full-size parity on sampled outputs: one Mamba-2.8B layer (d_model 2560, d_inner 5120,
dt_rank 160) in the launch configuration bench.py times (batch 16, the 2048-token prompt as
one prefill chunk, M = 32768 rows; then decode steps through the CUDA-graph-safe decode
path), checked against the fp64 oracle on sampled batch rows (the oracle computes a row in
seconds; rows are independent).  Also Falcon-Mamba-7B- and Zamba-7B-shaped
layers on shorter prompts."""
import numpy as np
import pytest
import torch

import synth
from oracle import mixer_ref as M
from paper_2602_21144_b200 import LayerWeights, State, TPMixer
from gpu_helpers import TOL, np64, prep_weights, rel

pytestmark = pytest.mark.gpu


def _run(dims, B, L, n_dec, rows, chunk=None):
    w = prep_weights(dims, 0, "bf16")
    g = torch.Generator().manual_seed(77)
    x = synth.bf16_round(torch.randn(B, L + n_dec, dims.d_model, generator=g, dtype=torch.float64))
    res = torch.randn(B, L + n_dec, dims.d_model, generator=g, dtype=torch.float64).float().double()
    mx = TPMixer(dims, "bf16")
    lw = LayerWeights(dims, w, dtype="bf16")
    st = State(mx, B)
    chunk = chunk or L
    outs = []
    for c0 in range(0, L, chunk):
        c = min(chunk, L - c0)
        xi = x[:, c0:c0 + c].to(torch.bfloat16).cuda().contiguous().view(B * c, -1)
        r = res[:, c0:c0 + c].float().cuda().contiguous().view(B * c, -1)
        mx.prefill(lw, st, xi, r, workspace=mx.workspace(B, c))
        outs.append(r.view(B, c, -1))
    wsd = mx.workspace(B, 1)
    for t in range(L, L + n_dec):
        xi = x[:, t].to(torch.bfloat16).cuda().contiguous()
        r = res[:, t].float().cuda().contiguous()
        mx.decode(lw, st, xi, r, workspace=wsd)
        outs.append(r.view(B, 1, -1))
    torch.cuda.synchronize()
    gpu = torch.cat([o.cpu() for o in outs], 1).double().numpy()
    h = st.h.cpu().double().numpy()
    wn = np64(w)
    for b in rows:
        ref, (_, h_ref) = M.mixer_forward(dims, wn, x[b:b + 1].numpy(), res[b:b + 1].numpy())
        d_gpu = gpu[b] - res[b].numpy()
        d_ref = ref[0] - res[b].numpy()
        assert rel(d_gpu[:L], d_ref[:L]) < TOL["bf16"], f"prefill row {b}"
        assert rel(d_gpu[L:], d_ref[L:]) < TOL["bf16"], f"decode row {b}"
        assert rel(h[b], h_ref[0]) < TOL["bf16"], f"state row {b}"


def test_mamba28b_layer_bench_config_sampled_rows():
    wl = synth.WORKLOADS["mamba2.8b"]
    _run(synth.CONFIGS["mamba2.8b"], wl["batch"], wl["prompt"], 3, rows=(0, wl["batch"] - 1))


def test_falcon7b_layer_chunked_sampled_rows():
    # Falcon-Mamba-7B shapes (d_model 4096, dt_rank 256, dt/B/C RMSNorm), chunked prefill
    _run(synth.CONFIGS["falcon7b"], 4, 512, 2, rows=(1,), chunk=192)


def test_zamba7b_layer_two_heads_sampled_rows():
    # Zamba-7B Mamba layer shapes (d_model 3712, dt_rank 232, 2 x_proj heads) at TP=1
    _run(synth.CONFIGS["zamba7b"], 4, 384, 2, rows=(2,))


def test_falcon7b_decode_bench_batch_sampled_rows():
    # the decode launch configuration bench.py times for Falcon-Mamba-7B: batch 32 through the
    # fused decode in_proj (P = 288 x_proj outputs per token) and the decode step
    _run(synth.CONFIGS["falcon7b"], synth.WORKLOADS["falcon7b"]["batch"], 64, 4, rows=(0, 31))


def test_zamba7b_decode_bench_batch_sampled_rows():
    _run(synth.CONFIGS["zamba7b"], synth.WORKLOADS["zamba7b"]["batch"], 64, 4, rows=(0, 15))
