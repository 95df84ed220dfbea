#!/usr/bin/env python
"""Per-layer decode time of a Mamba-shaped stack (graph-replayed, PDL) through
ssm_mixer_decode_block, plus the launch list of one step.

    python scripts/decode_layer_time.py [--config mamba2.8b] [--layers 16] [--batch 16] [--reps 20]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):   # same-box A/B of kernel variants (scripts/ab_build.sh)
    sys.path.insert(0, os.environ["DS_PKG_ROOT"])
import synth  # noqa: E402
from paper_2602_21144_b200 import LayerWeights, State, TPMixer, _lib as L  # noqa: E402
from paper_2602_21144_b200.stack import synthetic_layer  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--layers", type=int, default=16)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--config", default="mamba2.8b")
    p.add_argument("--unfused", action="store_true")
    a = p.parse_args()
    dims = synth.CONFIGS[a.config]
    B, nl = a.batch, a.layers
    mx = TPMixer(dims, "bf16")
    lws = [LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16").pack(mx) for l in range(nl)]
    sts = [State(mx, B) for _ in range(nl)]
    ws = mx.workspace(B, 1)
    res = torch.randn(B, dims.d_model, device="cuda")
    fl = L.SSM_AR2_INT8 | (L.SSM_DECODE_UNFUSED if a.unfused else 0)

    def step(s):
        for lw, st in zip(lws, sts):
            mx.decode_block(lw, st, res, 1e-5, fl, ws, s)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    before = mx.launches()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(torch.cuda.current_stream())
    nlaunch = mx.launches() - before
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / a.reps / nl
    print(f"{a.config} B={B} {'unfused' if a.unfused else 'fused'}: {us:7.2f} us/layer ({nlaunch / nl:.0f} launches/layer)",
          flush=True)


if __name__ == "__main__":
    main()
