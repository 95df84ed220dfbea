"""Per-kernel prefill timing of one Mamba-2.8B layer chunk (batch 16 x 2048 tokens) through the library's
CUDA-event probes (no profiler): in_proj, conv, x_proj, dt_proj, scan, out_proj.

    python scripts/prefill_time.py [--reps 5]
"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):   # same-box A/B of kernel variants
    sys.path.insert(0, os.environ["DS_PKG_ROOT"])
import synth  # noqa: E402
from paper_2602_21144_b200 import LayerWeights, TPMixer, _lib as L  # noqa: E402
from paper_2602_21144_b200.mixer import State  # noqa: E402
from paper_2602_21144_b200.stack import synthetic_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--config", default="mamba2.8b")
ap.add_argument("--pair", type=int, default=-1, help="CTA-pair GEMM mode (ssm_dbg_set_gemm_pair)")
args = ap.parse_args()
L.call("ssm_dbg_set_gemm_pair", args.pair)
dims = synth.CONFIGS[args.config]
wl = synth.WORKLOADS[args.config]
B, Lp = wl["batch"], wl["prompt"]
while B * Lp > 65536:
    Lp //= 2
mx = TPMixer(dims, "bf16")
lw = LayerWeights(dims, synthetic_layer(dims, 0), 1, 0, "bf16")
st = State(mx, B)
x = torch.randn(B * Lp, dims.d_model, device="cuda").to(torch.bfloat16)
r = torch.randn(B * Lp, dims.d_model, device="cuda")
ws = mx.workspace(B, Lp)
kinds = ["in_proj", "conv", "x_proj", "dt_proj", "scan", "out_proj"]
for k in kinds:
    mx.probe(k, args.reps + 2)
for _ in range(args.reps + 2):
    st.reset()
    mx.prefill(lw, st, x, r, L.SSM_AR2_INT8, ws)
torch.cuda.synchronize()
print(f"{args.config} prefill chunk: batch {B} x {Lp} tokens, one layer (median of {args.reps} after 2 warm-up), "
      f"gemm pair mode {args.pair}")
tot = 0.0
for k in kinds:
    ms = mx.probe_read(k)[2:]
    med = statistics.median(ms) * 1000 if ms else float("nan")
    tot += med if ms else 0.0
    print(f"  {k:9s} {med:8.1f} us")
print(f"  {'sum':9s} {tot:8.1f} us")
