#!/usr/bin/env python
"""Decode graph time per layer with DISTINCT weights per layer (the real case: every weight
byte streams from HBM) vs ONE weight set shared by all layers (weights stay L2-resident).
The gap bounds what moving the weight stream off the critical path (L2 prefetch) can win."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights, TPMixer  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mamba2.8b"
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 16
dims = synth.CONFIGS[cfg]
B = synth.WORKLOADS[cfg]["batch"]
mx = TPMixer(dims, "bf16")
for mode in ("distinct", "shared"):
    if mode == "distinct":
        layers = [LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16") for l in range(nl)]
    else:
        one = LayerWeights(dims, synthetic_layer(dims, 0), 1, 0, "bf16")
        layers = [one] * nl
    for lw in set(map(id, layers)):
        pass
    seen = set()
    for lw in layers:
        if id(lw) not in seen:
            lw.pack(mx)
            seen.add(id(lw))
    stack = MixerStack(mx, layers, B, 1)
    res = torch.randn(B, dims.d_model, device="cuda")
    g = stack.capture_decode(res)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 20 / nl
    print(f"{cfg} weights={mode:8s} pf={os.environ.get('SSM_DSTEP_PF', '0')} skip={os.environ.get('SSM_DEBUG_SKIP', '0')}: "
          f"{us:8.2f} us/layer", flush=True)
    del stack, g, layers
    torch.cuda.empty_cache()
