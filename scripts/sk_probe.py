#!/usr/bin/env python
"""Decode in_proj-shaped weight-streaming GEMM (M=16 tokens, W [10240 x 2560] pre-tiled) under
CUDA-graph replay: one CTA per 128-row tile (ksplit 1) vs split-K 2 vs stream-K over all SMs
(plain fp32 epilogues; the split variants include a 655 KB memset, timed separately)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import TPMixer  # noqa: E402

M, N, K = 16, 10240, 2560
mx = TPMixer(synth.CONFIGS["tiny"], "bf16")
copies = 8
W = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(copies)]
PK = [mx.pack_weight(w) for w in W]
X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda")


def timed(fn, reps=24):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps / 5


ms = timed(lambda i: C.zero_())
print(f"memset 655 KB: {ms:.2f} us")
for ks in (1, 2, 4, -1):
    t = timed(lambda i: mx.dbg_gemm_packed(X, W[i % copies], PK[i % copies], C, ksplit=ks))
    extra = ms if ks != 1 else 0.0
    print(f"ksplit {ks:3d}: {t:.2f} us/launch (minus memset {t - extra:.2f}) -> {N * K * 2 / (t - extra) / 1e3:.0f} GB/s")
