"""Decode-token latency of the full-depth stack: persistent whole-stack kernel vs the
per-layer kernel chain (both CUDA-graph replayed).  Usage: python scripts/stack_decode_time.py [config] [layers]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import _lib as L  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights, TPMixer  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mamba2.8b"
dims = synth.CONFIGS[cfg]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else dims.n_layers
B = int(os.environ.get("B", synth.WORKLOADS[cfg]["batch"]))
mx = TPMixer(dims, "bf16")
layers = []
for l in range(nl):
    full = synthetic_layer(dims, l)
    layers.append(LayerWeights(dims, full, 1, 0, "bf16").pack(mx))
    del full
torch.cuda.empty_cache()
res = torch.randn(B, dims.d_model, device="cuda")
for persistent in (True, False):
    st = MixerStack(mx, layers, B, 1, L.SSM_AR2_INT8, persistent=persistent)
    g = st.capture_decode(res, warmup=True)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    n = 50
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for e0, e1 in evs:
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    ms = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
    st.stack_check()
    med = ms[n // 2]
    if persistent:
        ring = [L.C.c_int32() for _ in range(3)] if hasattr(L, "C") else None
    print(f"{cfg} layers={nl} B={B} persistent={persistent}: median {med*1000:.1f} us/token "
          f"({med*1000/nl:.2f} us/layer), min {ms[0]*1000:.1f}, max {ms[-1]*1000:.1f}", flush=True)
    del st, g
