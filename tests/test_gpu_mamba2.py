"""GPU parity of the Mamba-2 (SSD) mixer through ssm_m2_mixer: chunked
prefill then decode from the cache, TP = 1 and virtual TP = 2 / 4 (heads split, B/C replicated,
norm statistics and out_proj all-reduced), against the fp64 oracle (oracle/mamba2_ref.py, pinned to
HF Mamba2Mixer), tolerance 2e-2 (bf16 I/O)."""
import numpy as np
import pytest
import torch

import synth
from oracle import mamba2_ref as M2
from paper_2602_21144_b200 import TPMixer, _lib as L
from paper_2602_21144_b200.mamba2 import Mamba2Mixer, Mamba2Weights
from gpu_helpers import TOL, VirtualGroup, rel

pytestmark = pytest.mark.gpu


def _run(m2, k, B, chunks, n_dec, flags, seed=9):
    D = m2.d_model
    T = sum(chunks) + n_dec
    w = synth.mamba2_weights(m2)
    g = torch.Generator().manual_seed(seed)
    x = synth.bf16_round(torch.randn(B, T, D, generator=g, dtype=torch.float64))
    res = torch.randn(B, T, D, generator=g, dtype=torch.float64).float().double()
    mdims = synth.MixerDims(d_model=D, d_inner=2 * D, dt_rank=max(16, D // 16))
    if k == 1:
        grp, mixers = None, [TPMixer(mdims, "bf16")]
    else:
        grp = VirtualGroup(mdims, k, "bf16", B * max(chunks))
        mixers = grp.mixers
    ws = [Mamba2Weights(m2, w, k, r) for r in range(k)]
    mix = [Mamba2Mixer(mixers[r], m2, B, max(chunks)) for r in range(k)]
    steps = [(int(t0), c) for t0, c in zip(np.cumsum([0] + chunks[:-1]), chunks)] + \
            [(sum(chunks) + j, 1) for j in range(n_dec)]
    outs = [[] for _ in range(k)]
    for t0, c in steps:
        xs = [x[:, t0:t0 + c].to(torch.bfloat16).cuda().contiguous().view(B * c, D) for _ in range(k)]
        rs = [res[:, t0:t0 + c].float().cuda().contiguous().view(B * c, D) for _ in range(k)]
        torch.cuda.synchronize()
        if grp is None:
            mix[0](ws[0], xs[0], rs[0], c, flags)
            torch.cuda.synchronize()
        else:
            grp.run(lambda r, mx, s: mix[r](ws[r], xs[r], rs[r], c, flags, s))
        for r in range(k):
            outs[r].append(rs[r].view(B, c, D).cpu())
    got = [torch.cat(o, 1).double().numpy() for o in outs]
    wq = {kk: (synth.bf16_round(v) if kk in ("w_in", "w_out") else v.float().double()).numpy() for kk, v in w.items()}
    ref, (_, h_ref) = M2.mixer_forward(m2, wq, x.numpy(), res.numpy())
    return got, ref, res.numpy(), mix, h_ref


@pytest.mark.parametrize("m2", [synth.Mamba2Dims(d_model=128, d_inner=256, d_state=16),
                                synth.Mamba2Dims(d_model=256, d_inner=512, d_state=128)])
def test_mamba2_tp1_prefill_decode_vs_oracle(m2):
    got, ref, res, mix, h_ref = _run(m2, 1, 2, [37, 20], 4, L.SSM_AR2_INT8)
    assert rel(got[0] - res, ref - res) < TOL["bf16"]
    H, P, N = m2.n_heads, m2.headdim, m2.d_state
    h = mix[0].h.view(2, H, P, N).cpu().double().numpy()
    assert rel(h, h_ref) < TOL["bf16"]


@pytest.mark.parametrize("k,flags", [(2, L.SSM_AR2_FP32), (4, L.SSM_AR2_FP32), (2, L.SSM_AR2_INT8)])
def test_mamba2_virtual_tp_vs_oracle(k, flags):
    m2 = synth.Mamba2Dims(d_model=256, d_inner=512, d_state=128)
    got, ref, res, _, _ = _run(m2, k, 2, [33, 31], 3, flags)
    for r in range(1, k):
        np.testing.assert_array_equal(got[r], got[0])
    assert rel(got[0] - res, ref - res) < TOL["bf16"]


def test_mamba2_2p7b_layer_shape():
    """The Mamba-2 2.7B layer shape (d_model 2560, 80 heads of 64, d_state 128), short prompt."""
    got, ref, res, _, _ = _run(synth.MAMBA2_2P7B, 1, 1, [48], 2, L.SSM_AR2_INT8)
    assert rel(got[0] - res, ref - res) < TOL["bf16"]


@pytest.mark.parametrize("N,B", [(16, 3), (64, 5), (128, 2)])
def test_mamba2_decode_step_alone_vs_oracle(N, B):
    """The L = 1 decode step (m2_scan_step: one lane group per state row) judged on the generated
    tokens alone, after a prompt long enough that the state carries the history; d_state 16/64/128
    (2 / 8 / 16 lanes per row), ragged batch."""
    m2 = synth.Mamba2Dims(d_model=256, d_inner=512, d_state=N)
    n_dec = 6
    got, ref, res, mix, h_ref = _run(m2, 1, B, [29], n_dec, L.SSM_AR2_INT8)
    dec = slice(29, 29 + n_dec)
    assert rel(got[0][:, dec] - res[:, dec], ref[:, dec] - res[:, dec]) < TOL["bf16"]
    H, P = m2.n_heads, m2.headdim
    assert rel(mix[0].h.view(B, H, P, N).cpu().double().numpy(), h_ref) < TOL["bf16"]


@pytest.mark.parametrize("N", [64, 128])
def test_mamba2_chunked_ssd_multi_chunk_vs_oracle(N):
    """Prompts longer than one 64-token SSD chunk, split across calls at chunk-unaligned offsets
    (150 = 2 x 64 + 22, then 70 carried from the saved state), so the chunk carry h_end, the
    in-chunk decay masks, the padded tail and the cross-call state all count."""
    m2 = synth.Mamba2Dims(d_model=256, d_inner=512, d_state=N)
    got, ref, res, mix, h_ref = _run(m2, 1, 2, [150, 70], 3, L.SSM_AR2_INT8)
    assert rel(got[0] - res, ref - res) < TOL["bf16"]
    H, P = m2.n_heads, m2.headdim
    assert rel(mix[0].h.view(2, H, P, N).cpu().double().numpy(), h_ref) < TOL["bf16"]


def test_mamba2_short_calls_per_token_scan_vs_oracle():
    """Calls shorter than 16 tokens take the per-token recurrence (m2_scan), not the chunked form."""
    m2 = synth.Mamba2Dims(d_model=256, d_inner=512, d_state=128)
    got, ref, res, _, _ = _run(m2, 1, 3, [7, 5, 13], 2, L.SSM_AR2_INT8)
    assert rel(got[0] - res, ref - res) < TOL["bf16"]


@pytest.mark.parametrize("k", [2, 4])
def test_mamba2_virtual_tp_multi_chunk_vs_oracle(k):
    """Virtual TP with prompts spanning several 64-token SSD chunks (chunk-unaligned, two calls), so
    each rank's chunked scan, its partial sums of squares and their all-reduce before the row-scaled
    out_proj all count; replicas must stay bitwise equal."""
    m2 = synth.Mamba2Dims(d_model=256, d_inner=512, d_state=128)
    got, ref, res, _, _ = _run(m2, k, 2, [97, 70], 3, L.SSM_AR2_FP32)
    for r in range(1, k):
        np.testing.assert_array_equal(got[r], got[0])
    assert rel(got[0] - res, ref - res) < TOL["bf16"]
