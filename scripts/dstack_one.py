"""One persistent whole-stack decode launch at the bench's Mamba-2.8B shape (for ncu captures).

    python scripts/dstack_one.py [--layers 64] [--calls 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import LayerWeights, TPMixer, _lib as L  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=64)
ap.add_argument("--calls", type=int, default=3)
args = ap.parse_args()
dims = synth.CONFIGS["mamba2.8b"]
B = synth.WORKLOADS["mamba2.8b"]["batch"]
mx = TPMixer(dims, "bf16")
layers = [LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16") for l in range(args.layers)]
stack = MixerStack(mx, layers, B, 16, L.SSM_AR2_INT8).persistent()
r = torch.randn(B, dims.d_model, device="cuda")
for _ in range(args.calls):
    stack.decode_step(r)
torch.cuda.synchronize()
print("ok")
