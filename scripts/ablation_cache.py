#!/usr/bin/env python
"""Caching ablation (§5.5, fig:ablation_latency: "Sharding" vs "Sharding +
Caching"): per-token decode latency WITH the SSM state cache (CUDA-graph decode step reading the
carried conv window and h) vs WITHOUT it (every new token re-runs prefill over the prompt plus
all tokens generated so far, the no-cache rescan arm).  TP=1 on one B200, Mamba-2.8B shapes,
256-token input and 256-token output as in the paper's ablation.  The rescan cost is measured at
sampled output positions and averaged over all 256 by the trapezoid rule (it grows linearly).
    python scripts/ablation_cache.py [--layers 64] [--batch 16] [--prompt 256] [--out 256]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights, TPMixer  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="mamba2.8b")
p.add_argument("--layers", type=int, default=64)
p.add_argument("--batch", type=int, default=16)
p.add_argument("--prompt", type=int, default=256)
p.add_argument("--out", type=int, default=256)
a = p.parse_args()
dims = synth.CONFIGS[a.config]
B, Lp, Lo, D = a.batch, a.prompt, a.out, dims.d_model
mx = TPMixer(dims, "bf16")
layers = []
for l in range(a.layers):
    lw = LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16")
    lw.pack(mx)
    layers.append(lw)
stack = MixerStack(mx, layers, B, Lp + Lo)
g = torch.Generator(device="cuda").manual_seed(42)
x_all = torch.randn(B, Lp + Lo, D, generator=g, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

# with cache: prefill the prompt once, then graph-replayed decode steps
res_t = torch.empty(B, D, device="cuda")
stack.reset()
pre = x_all[:, :Lp].reshape(B * Lp, D).contiguous()
stack.prefill_chunk(pre)
graph = stack.capture_decode(res_t)
stack.reset()
pre = x_all[:, :Lp].reshape(B * Lp, D).contiguous()
stack.prefill_chunk(pre)
torch.cuda.synchronize()
e0.record()
for j in range(Lo):
    res_t.copy_(x_all[:, Lp + j])
    graph.replay()
e1.record()
torch.cuda.synchronize()
cached_ms = e0.elapsed_time(e1) / Lo


# without cache: token j costs a prefill over Lp + j + 1 tokens from a zero state
def rescan_ms(n):
    buf = x_all[:, :n].reshape(B * n, D).contiguous()
    stack.reset()
    stack.prefill_chunk(buf.clone())           # warm
    ts = []
    for _ in range(2):
        w = buf.clone()
        stack.reset()
        torch.cuda.synchronize()
        e0.record()
        stack.prefill_chunk(w)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


pos = sorted(set([0, Lo // 4, Lo // 2, 3 * Lo // 4, Lo - 1]))
samples = [(j, rescan_ms(Lp + j + 1)) for j in pos]
tot = 0.0
for (j0, t0), (j1, t1) in zip(samples[:-1], samples[1:]):
    tot += (t0 + t1) / 2 * (j1 - j0)
rescan_avg = (tot + samples[0][1]) / Lo
print(json.dumps(dict(config=a.config, layers=a.layers, batch=B, prompt=Lp, out=Lo, tp=1,
                      per_token_ms_with_cache=cached_ms, per_token_ms_rescan=rescan_avg,
                      rescan_samples_ms={str(j): t for j, t in samples}, speedup=rescan_avg / cached_ms)))
