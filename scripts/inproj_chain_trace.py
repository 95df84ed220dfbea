#!/usr/bin/env python
"""Per-CTA pipeline timeline of the fused decode in_proj INSIDE the graph-replayed decode chain
(GPU only).  Run with SSM_GEMM_NOMMA=8 (trace slots on) and SSM_DEBUG_SKIP=16 (no out_proj, so the
last GEMM launch of a replay -- whose trace survives -- is the last layer's in_proj).  Prints the
event offsets (us from each CTA's entry) for x-tile CTAs (conv + x_proj epilogue) and z-tile CTAs."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import _lib as L  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights, TPMixer  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402

NAMES = ["gt_entry", "clk_entry", "prologue_done", "tma_first_issue", "mma_first_full", "mma_last_full",
         "mma_done_commit", "epi_tfull", "epi_tmem_ld", "epi_stores_done", "cta_end_sync", "dealloc_done",
         "gt_exit"]
dims = synth.CONFIGS["mamba2.8b"]
B, nl = 16, 8
mx = TPMixer(dims, "bf16")
layers = []
for l in range(nl):
    lw = LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16")
    lw.pack(mx)
    layers.append(lw)
stack = MixerStack(mx, layers, B, 1)
res = torch.randn(B, dims.d_model, device="cuda")
g = stack.capture_decode(res)
for _ in range(4):
    g.replay()
torch.cuda.synchronize()
ctas = 2 * dims.d_inner // 128
buf = (ctypes.c_uint64 * (1024 * 16))()
L.call("ssm_dbg_gemm_trace", buf, 1024 * 16)
t = np.array(buf[:ctas * 16], dtype=np.float64).reshape(ctas, 16)
ghz = 1.965
gt0 = t[:, 0].min()
print(f"fused decode in_proj in the chain: {ctas} CTAs (x-tiles 0..{ctas // 2 - 1}, z-tiles {ctas // 2}..{ctas - 1})")
for name, sel in (("x-tiles", slice(0, ctas // 2)), ("z-tiles", slice(ctas // 2, ctas))):
    print(f" {name}: entry spread {(t[sel, 0].max() - t[sel, 0].min()) / 1000:.2f} us, exit (gt) min "
          f"{(t[sel, 12].min() - gt0) / 1000:.2f} med {(np.median(t[sel, 12]) - gt0) / 1000:.2f} max {(t[sel, 12].max() - gt0) / 1000:.2f} us after the first entry")
    for j in range(2, 12):
        v = t[sel, j] / ghz / 1000
        print(f"   {NAMES[j]:16s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
