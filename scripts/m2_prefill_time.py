#!/usr/bin/env python
"""Prefill time of one Mamba-2-2.7B mixer layer (batch 16 x 2048 tokens, SSD chunk path) by CUDA events,
median of --reps calls after two warm-up calls (GPU only).  Honours DS_PKG_ROOT for same-box A/B builds.
    python scripts/m2_prefill_time.py [--reps 5]"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):
    sys.path.insert(0, os.environ["DS_PKG_ROOT"])
import synth  # noqa: E402
from paper_2602_21144_b200 import TPMixer  # noqa: E402
from paper_2602_21144_b200.mamba2 import Mamba2Mixer, Mamba2Weights, synthetic_mamba2_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--seqlen", type=int, default=2048)
a = ap.parse_args()
m2 = synth.MAMBA2_2P7B
dims = synth.CONFIGS["mamba2.8b"]
B, Lp = a.batch, a.seqlen
mx = TPMixer(dims, "bf16")
w = Mamba2Weights(m2, synthetic_mamba2_layer(m2, 0, device="cuda"), 1, 0, "cuda")
mix = Mamba2Mixer(mx, m2, B, Lp)
x = torch.randn(B * Lp, dims.d_model, device="cuda").to(torch.bfloat16)
r = torch.randn(B * Lp, dims.d_model, device="cuda")
ts = []
for i in range(a.reps + 2):
    mix.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mix(w, x, r, Lp)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1) * 1000)
print(f"Mamba-2-2.7B layer prefill, batch {B} x {Lp}: {statistics.median(ts):.1f} us (median of {a.reps})")
