"""Timeline of the persistent whole-stack decode (ssm_dbg_dstack_trace): per-phase durations per
layer, medians / maxima over CTAs, at the bench's Mamba-2.8B shape (batch 16).

    python scripts/dstack_trace.py [--layers 64] [--prompt 64] [--ctas 0]
"""
import argparse
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("DS_PKG_ROOT"):   # same-box A/B of kernel variants (scripts/ab_build.sh)
    sys.path.insert(0, os.environ["DS_PKG_ROOT"])
import synth  # noqa: E402
from paper_2602_21144_b200 import LayerWeights, TPMixer, _lib as L  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=64)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--config", default="mamba2.8b")
    args = ap.parse_args()
    dims = synth.CONFIGS[args.config]
    B = synth.WORKLOADS[args.config]["batch"]
    nl = args.layers
    mx = TPMixer(dims, "bf16")
    layers = []
    for l in range(nl):
        f = synthetic_layer(dims, l)
        layers.append(LayerWeights(dims, f, 1, 0, "bf16"))
        del f
    stack = MixerStack(mx, layers, B, args.prompt, L.SSM_AR2_INT8).persistent(args.ctas)
    res = torch.randn(B * args.prompt, dims.d_model, device="cuda")
    stack.prefill_chunk(res)
    r = torch.randn(B, dims.d_model, device="cuda")
    for _ in range(5):
        stack.decode_step(r)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        stack.decode_step(r)
    ev[1].record()
    torch.cuda.synchronize()
    tok_ms = ev[0].elapsed_time(ev[1]) / 10
    nc = args.ctas or torch.cuda.get_device_properties(0).multi_processor_count
    tr = torch.zeros(nc * nl * 32, dtype=torch.int64, device="cuda")
    L.call("ssm_dbg_dstack_trace", stack.dstack.handle, C.c_void_p(tr.data_ptr()))
    stack.decode_step(r)
    torch.cuda.synchronize()
    L.call("ssm_dbg_dstack_trace", stack.dstack.handle, C.c_void_p(0))
    t = tr.view(nc, nl, 32).cpu().double()
    print(f"{args.config}: {nl} layers, batch {B}, {nc} CTAs: {tok_ms * 1000:.1f} us/token untraced "
          f"({tok_ms * 1000 / nl:.2f} us/layer)")
    names = ["A mma", "A epi", "bar A", "B", "B loads", "B mbB", "B dt", "B items", "bar B", "C mma", "C epi", "bar C",
             "layer"]
    rows = {n: [] for n in names}
    waits = {"A wait": [], "C wait": []}
    for l in range(2, nl - 1):
        s = t[:, l]
        s0 = s[:, 0]
        a_end = torch.maximum(s[:, 1], s[:, 2])
        c_end = torch.maximum(s[:, 6], s[:, 7])
        vals = {"A mma": s[:, 1] - s0, "A epi": s[:, 2] - s0, "bar A": s[:, 3] - a_end, "B": s[:, 4] - s[:, 3],
                "B loads": s[:, 11] - s[:, 3], "B mbB": s[:, 12] - s[:, 11], "B dt": s[:, 13] - s[:, 12],
                "B items": s[:, 4] - s[:, 13],
                "bar B": s[:, 5] - s[:, 4], "C mma": s[:, 6] - s[:, 5], "C epi": s[:, 7] - s[:, 5],
                "bar C": s[:, 8] - c_end, "layer": s[:, 8] - s0}
        for k, v in vals.items():
            rows[k].append((float(v.median()), float(v.max()), float(v.min())))
        pass

    print(f"{'phase':8s} {'median us':>10s} {'max us':>10s} {'min us':>10s}   (medians over layers 2..{nl - 2})")
    for k in names:
        med = statistics.median(x[0] for x in rows[k]) / 1000
        mx_ = statistics.median(x[1] for x in rows[k]) / 1000
        mn = statistics.median(x[2] for x in rows[k]) / 1000
        print(f"{k:8s} {med:10.2f} {mx_:10.2f} {mn:10.2f}")
    # epilogue progress over phase A's units (CTA 0, layer 10): unit i started / partials ready, us
    l = min(10, nl - 2)
    s = t[0, l]
    print("A epi units (CTA 0, layer %d): " % l + "  ".join(
        f"{(s[16 + i] - s[0]) / 1000:.2f}/{(s[24 + i] - s[0]) / 1000:.2f}" for i in range(8) if s[16 + i] > 0))
    if os.environ.get("DS_FINE"):   # fine stamps inside unit 2 of phase A (a variant built for it)
        for cc in (0, 50, 100):
            s = t[cc, 10]
            print(f"CTA {cc} unit 2: " + "  ".join(f"{k}:{(s[k] - s[16]) / 1000:.2f}" for k in range(16, 23)))
    if os.environ.get("DS_FINE2"):  # MMA warp 0: unit i wait-start / data-landed (last layer; variant build)
        for cc in (0, 50, 100):
            s = t[cc, nl - 1]
            print(f"CTA {cc} A units (wait/landed, us from layer start): " + "  ".join(
                f"{(s[16 + i] - s[0]) / 1000:.2f}/{(s[24 + i] - s[0]) / 1000:.2f}" for i in range(8) if s[16 + i] > 0))
    if os.environ.get("DS_FINE3"):  # MMA warps 0 / kMW-1, units 0-3 of phase A: wait-full, mma, wait-free (ns)
        for cc in (0, 70, 140):
            s = tr.view(nc, nl, 32)[cc, nl - 1].cpu()
            parts = []
            for w in (0, 1):
                for i in range(4):
                    v0, v1 = int(s[16 + 8 * w + 2 * i]), int(s[17 + 8 * w + 2 * i])
                    parts.append(f"w{w}u{i}:{(v0 >> 32)}/{v0 & 0xffffffff}/{v1}")
            print(f"CTA {cc}: " + " ".join(parts))
    # layer-to-layer: start of layer l+1 - start of layer l, min over CTAs
    st = t[:, :, 0]
    d = (st[:, 3:nl - 1] - st[:, 2:nl - 2]).median(0).values
    print(f"layer period (median CTA): {float(d.median()) / 1000:.2f} us")


if __name__ == "__main__":
    main()
