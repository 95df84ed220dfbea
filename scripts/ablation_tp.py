#!/usr/bin/env python
"""The structure of the paper's ablation (fig:ablation_latency: "Sharding",
"+ Caching", "+ Quantization") plus the naive four-collective sharding of §4.2,
as per-token latency of a Mamba-2.8B-shaped stack at TP = k on ONE B200 (k virtual ranks: the
same peer-to-peer kernels and flag protocol, but the ranks share one GPU's SMs and HBM, so the
absolute numbers are one device doing all ranks' work -- only the arms' ordering and ratios carry
over, NVLink costs do not).

Arms (256-token input, 256-token output, as in the paper's ablation):
  naive_rescan    naive sharding (2 all-gathers + 2 all-reduces per block), no SSM cache: every
                  new token re-runs prefill over prompt + generated tokens
  split_rescan    channel splitter (2 all-reduces per block), no cache
  split_cache     channel splitter + SSM cache (graph-replayed decode step), exact fp32 AR#2
  split_cache_q   + int8 quantised AR#2
The rescan cost grows linearly with the prefix, so it is sampled at 5 output positions and
averaged by the trapezoid rule.
    python scripts/ablation_tp.py [--tp 2] [--layers 64] [--batch 1] [--prompt 256] [--out 256]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import _lib as L  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402
from paper_2602_21144_b200.virtual import VirtualGroup  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="mamba2.8b")
p.add_argument("--tp", type=int, default=2)
p.add_argument("--layers", type=int, default=64)
p.add_argument("--batch", type=int, default=1)
p.add_argument("--prompt", type=int, default=256)
p.add_argument("--out", type=int, default=256)
p.add_argument("--arms", default="naive_rescan,split_rescan,split_cache,split_cache_q")
a = p.parse_args()
dims = synth.CONFIGS[a.config]
k, B, Lp, Lo, D = a.tp, a.batch, a.prompt, a.out, dims.d_model
Lmax = Lp + Lo
g = torch.Generator(device="cuda").manual_seed(42)
x_all = torch.randn(B, Lmax, D, generator=g, device="cuda")
fulls = [synthetic_layer(dims, l) for l in range(a.layers)]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def build(flags, naive):
    grp = VirtualGroup(dims, k, "bf16", B * Lmax)
    stacks = []
    for r in range(k):
        lws = [LayerWeights(dims, f, k, r, "bf16", naive=naive).pack(grp.mixers[r]) for f in fulls]
        stacks.append(MixerStack(grp.mixers[r], lws, B, Lmax, flags))
    torch.cuda.synchronize()
    return grp, stacks


def timed(grp, fn):
    torch.cuda.synchronize()
    e0.record()
    grp.run(fn)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def rescan_avg(grp, stacks):
    def one(n):
        bufs = [x_all[:, :n].reshape(B * n, D).contiguous() for _ in range(k)]
        grp.run(lambda r, mx, s: (stacks[r].reset(s), stacks[r].prefill_chunk(bufs[r].clone(), s)))   # warm
        ts = []
        for _ in range(2):
            ws = [b.clone() for b in bufs]
            ts.append(timed(grp, lambda r, mx, s: (stacks[r].reset(s), stacks[r].prefill_chunk(ws[r], s))))
        return min(ts)
    pos = sorted(set([0, Lo // 4, Lo // 2, 3 * Lo // 4, Lo - 1]))
    samples = [(j, one(Lp + j + 1)) for j in pos]
    tot = 0.0
    for (j0, t0), (j1, t1) in zip(samples[:-1], samples[1:]):
        tot += (t0 + t1) / 2 * (j1 - j0)
    return (tot + samples[0][1]) / Lo, samples


def cached_avg(grp, stacks):
    rts = [torch.empty(B, D, device="cuda") for _ in range(k)]
    pre = [x_all[:, :Lp].reshape(B * Lp, D).contiguous() for _ in range(k)]
    grp.run(lambda r, mx, s: (stacks[r].reset(s), stacks[r].prefill_chunk(pre[r].clone(), s)))
    graphs = []
    for r in range(k):
        with torch.cuda.stream(grp.streams[r]):
            graphs.append(stacks[r].capture_decode(rts[r], warmup=False))
    grp.run(lambda r, mx, s: (stacks[r].reset(s), stacks[r].prefill_chunk(pre[r].clone(), s)))
    ms = []
    for j in range(Lo):
        for r in range(k):
            rts[r].copy_(x_all[:, Lp + j])
        ms.append(timed(grp, lambda r, mx, s: stacks[r].replay(graphs[r], s)))
    return sum(ms[8:]) / max(len(ms) - 8, 1)


out = dict(config=a.config, layers=a.layers, tp=k, batch=B, prompt=Lp, out=Lo, virtual_ranks_on_one_gpu=True)
arms = {"naive_rescan": (L.SSM_AR2_FP32 | L.SSM_TP_NAIVE, True, "rescan"),
        "split_rescan": (L.SSM_AR2_FP32, False, "rescan"),
        "split_cache": (L.SSM_AR2_FP32, False, "cache"),
        "split_cache_q": (L.SSM_AR2_INT8, False, "cache")}
for name in a.arms.split(","):
    flags, naive, kind = arms[name]
    grp, stacks = build(flags, naive)
    if kind == "rescan":
        avg, samples = rescan_avg(grp, stacks)
        out[name] = dict(per_token_ms=avg, samples_ms={str(j): t for j, t in samples})
    else:
        out[name] = dict(per_token_ms=cached_avg(grp, stacks))
    print(name, json.dumps(out[name]), flush=True)
    del grp, stacks
    torch.cuda.empty_cache()
print(json.dumps(out))
