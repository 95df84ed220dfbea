#!/usr/bin/env python
"""Per-kernel device time of the decode step (GPU only): eager decode (so kernels do not
overlap) with the library's CUDA-event probes around each kernel kind, Mamba-2.8B shapes,
batch 16, weights of `--layers` layers rotating so they stream from HBM as in real decode."""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights, TPMixer  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="mamba2.8b")
    p.add_argument("--layers", type=int, default=8)
    p.add_argument("--steps", type=int, default=6)
    a = p.parse_args()
    dims = synth.CONFIGS[a.config]
    B = synth.WORKLOADS[a.config]["batch"]
    mx = TPMixer(dims, "bf16")
    layers = [LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16") for l in range(a.layers)]
    stack = MixerStack(mx, layers, B, 1)
    res = torch.randn(B, dims.d_model, device="cuda")
    for _ in range(2):
        stack.decode_step(res)
    torch.cuda.synchronize()
    out = {}
    for kind in ["in_proj", "conv", "x_proj", "decode_step", "out_proj"]:
        mx.probe(kind, a.layers * a.steps + 8)
        for _ in range(a.steps):
            stack.decode_step(res)
        torch.cuda.synchronize()
        ms = mx.probe_read(kind)
        mx.probe(kind, 0)
        out[kind] = statistics.median(ms) * 1000
    # rmsnorm (separate ABI call) timed with torch events
    x = torch.empty(B, dims.d_model, device="cuda", dtype=torch.bfloat16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        e0.record()
        mx.rmsnorm(res, x)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    out["rmsnorm"] = statistics.median(ts)
    # whole decode step in a CUDA graph
    g = stack.capture_decode(res)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    step_us = e0.elapsed_time(e1) * 1000 / 10 / a.layers
    tot = sum(out.values())
    for k, v in out.items():
        print(f"{a.config} decode {k:12s} {v:8.2f} us")
    print(f"{a.config} decode sum of kernels {tot:8.2f} us/layer; graph replay {step_us:8.2f} us/layer "
          f"(launch gaps ~{(step_us - tot):.2f} us/layer)")


if __name__ == "__main__":
    main()
