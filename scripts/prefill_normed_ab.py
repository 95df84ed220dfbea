"""Same-process A/B of the stack prefill with the pre-norm folded into the projections
(ssm_mixer_prefill_normed) against rmsnorm + ssm_mixer_prefill: Mamba-2.8B, batch 16 x 2048, 64 layers.

    python scripts/prefill_normed_ab.py [--layers 64] [--reps 3]
"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import LayerWeights, TPMixer, _lib as L  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
dims = synth.CONFIGS["mamba2.8b"]
B, Lp = 16, 2048
mx = TPMixer(dims, "bf16")
layers = [LayerWeights(dims, synthetic_layer(dims, l % 8), 1, 0, "bf16") for l in range(args.layers)]
stack = MixerStack(mx, layers, B, Lp, L.SSM_AR2_INT8)
x0 = torch.randn(B * Lp, dims.d_model, device="cuda")
res = torch.empty_like(x0)
out = {}
for mode in (True, False, True, False):
    stack.prefill_normed = mode
    ts = []
    for _ in range(args.reps + 1):
        stack.reset()
        res.copy_(x0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        stack.prefill_chunk(res)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out.setdefault(mode, []).append(statistics.median(ts[1:]))
    if mode:
        r_normed = res.clone()
    else:
        diff = (res - r_normed).abs().max().item() / (res - x0).abs().max().item()
for mode, v in out.items():
    print(f"prefill_normed={mode}: {' / '.join(f'{t:.2f}' for t in v)} ms for {args.layers} layers")
print(f"max |difference| of the residual update between the two paths, relative: {diff:.2e}")
