#!/usr/bin/env python
"""Decode-step graph replay time per layer (GPU only).  Run under different
SSM_DEBUG_SKIP / SSM_DEBUG_SKIP_NORM settings to get each kernel's marginal cost."""
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
layers = [LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16") for l in range(nl)]
if os.environ.get("SSM_ABL_PACK", "1") == "1":
    for lw in layers:
        lw.pack(mx)
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
print(f"{cfg} skip={os.environ.get('SSM_DEBUG_SKIP', '0')} skipnorm={os.environ.get('SSM_DEBUG_SKIP_NORM', '0')} "
      f"pdl={os.environ.get('SSM_PDL', '1')} pack={os.environ.get('SSM_ABL_PACK', '1')}: {us:8.2f} us/layer  kernels/step={stack.graph_launches}", flush=True)
