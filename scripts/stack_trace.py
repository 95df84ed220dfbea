"""Timeline of the persistent decode kernel (ssm_dbg_stack_trace): per-phase durations and
barrier waits, medians over CTAs and layers.  Usage: python scripts/stack_trace.py [config] [layers]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import _lib as L  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights, TPMixer  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mamba2.8b"
dims = synth.CONFIGS[cfg]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 16
B = int(os.environ.get("B", synth.WORKLOADS[cfg]["batch"]))
mx = TPMixer(dims, "bf16")
layers = [LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16").pack(mx) for l in range(nl)]
st = MixerStack(mx, layers, B, 1, L.SSM_AR2_INT8, persistent=True)
G = torch.cuda.get_device_properties(0).multi_processor_count
tr = torch.zeros(G * nl * 32, dtype=torch.int64, device="cuda")
res = torch.randn(B, dims.d_model, device="cuda")
for _ in range(3):
    st.decode_step(res)
L.call("ssm_dbg_stack_trace", mx.handle, C.c_void_p(tr.data_ptr()), tr.numel() * 8)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st.decode_step(res)
e1.record()
torch.cuda.synchronize()
L.call("ssm_dbg_stack_trace", mx.handle, None, 0)
st.stack_check()
t = tr.view(G, nl, 32).cpu().numpy().astype(np.float64)
acc = t.copy()
ri, gr, cpc = C.c_int32(), C.c_int32(), C.c_int32()
L.call("ssm_stack_info", mx.handle, C.byref(ri), C.byref(gr), C.byref(cpc))
print(f"ring slots {ri.value}, grid {gr.value}, channels/CTA <= {cpc.value}")
t0 = t[:, 0, 0].min()
t = (t - t0) / 1000.0  # us

print(f"{cfg} layers={nl} B={B}: launch {e0.elapsed_time(e1)*1000:.1f} us, first stamp->last layer end "
      f"{t[:, -1, 8].max():.1f} us")
names = [(0, 1, "A prologue"), (1, 2, "A in_proj (epilogue drained)"), (2, 3, "A barrier"),
         (3, 16, "B loads + rs"), (16, 17, "B conv items"), (17, 4, "B x_proj mma"), (4, 5, "B barrier"),
         (5, 18, "C dbc load"), (18, 19, "C dt prep + mma"), (19, 6, "C scan items"), (6, 7, "C barrier"),
         (7, 8, "D out_proj + finalise"), (8, 9, "D barrier")]
lay = slice(1, nl)  # skip layer 0 (ramp)
for a, b, nm in names:
    d = t[:, lay, b] - t[:, lay, a]
    print(f"  {nm:34s} median {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f} us")
per_layer = np.diff(t[0, :, 0])
print(f"  layer period (CTA 0): median {np.median(per_layer):.2f} us")
# producer: layer start (12) and W_out start (13) relative to the consumers' phase A start
lead = t[:, lay, 0] - t[:, lay, 12]
print(f"  producer lead at layer start (consumer A start - producer layer start): median {np.median(lead):.2f} us")
win = t[:, lay, 13] - t[:, lay, 12]
print(f"  producer time issuing W_in units: median {np.median(win):.2f} us")
def med(a, b):
    d = [t[:, l, b] - t[:, l, a] for l in range(1, nl - 1)]
    return np.median(np.concatenate(d))
print("  A: start(1)->B staged(23) %.2f, ->MMA first unit(24) %.2f, MMA first->last(24->25) %.2f, last->drained(25->2) %.2f"
      % (med(1, 23), med(1, 24), med(24, 25), med(25, 2)))
print("  D: start(7)->B staged(22) %.2f, ->MMA first unit(20) %.2f, MMA first->last(20->21) %.2f, last->D end(21->8) %.2f"
      % (med(7, 22), med(7, 20), med(20, 21), med(21, 8)))
for k, nm in ((30, "A: MMA wait weights"), (31, "A: MMA wait B"), (26, "D: MMA wait weights"), (27, "D: MMA wait B")):
    d = acc[:, 1:, k] / 1965.0
    print(f"  {nm:24s} median {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f} us (clock64 @1.965GHz)")
for k, nm in ((10, "A: MMA issue (elected lane)"), (11, "A: issue+commit+syncwarp"), (14, "A: MMA loop total")):
    d = acc[:, 1:, k] / 1965.0
    print(f"  {nm:28s} median {np.median(d):7.2f} us (clock64)")
print("  A staging bempty waits: %.2f us (clock64), failed try_waits median %d" % (np.median(acc[:, 1:, 28]) / 1965.0, np.median(acc[:, 1:, 29])))
