#!/usr/bin/env python
"""Per-kernel roofline table for every §8(a) row (GPU only): Mamba-2.8B shapes, batch 16,
prompt 2048 (one chunk) and single-token decode, TP=1.  Each kernel kind is timed by the
library's CUDA-event probes (eager launches, weights of `--layers` distinct layers so they
stream from HBM), and its ALGORITHMIC work -- SURVEY.md §8(d) per-unit figures x the units one
launch processes -- is divided by the median launch time and by the binding peak
(MEASURED_PEAKS.json: hbm_gbs, bf16_tflops -- the burst figure: each GEMM runs ~1 ms at full clock; MUFU from the guide's unit count:
16 ex2/clk/SM x 148 SMs x the max SM clock).
    python scripts/kernel_rooflines.py [--layers 8] [--json out.json]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2602_21144_b200.mixer import LayerWeights, TPMixer  # noqa: E402
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="mamba2.8b")
    p.add_argument("--layers", type=int, default=8)
    p.add_argument("--json", default="")
    a = p.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"] * 1e9
    tc = peaks["bf16_tflops"] * 1e12
    mufu = 16 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6  # ex2 per second
    dims = synth.CONFIGS[a.config]
    wl = synth.WORKLOADS[a.config]
    B, Lp = wl["batch"], wl["prompt"]
    while B * Lp > 65536:
        Lp //= 2
    D, E, N, R = dims.d_model, dims.d_inner, dims.d_state, dims.dt_rank
    P = R + 2 * N
    M = B * Lp
    mx = TPMixer(dims, "bf16")
    layers = []
    for l in range(a.layers):
        lw = LayerWeights(dims, synthetic_layer(dims, l), 1, 0, "bf16")
        lw.pack(mx)
        layers.append(lw)
    stack = MixerStack(mx, layers, B, Lp)
    g = torch.Generator(device="cuda").manual_seed(42)
    x0 = torch.randn((M, D), generator=g, device="cuda")
    res = x0.clone()
    stack.reset()
    stack.prefill_chunk(res)   # warm-up (allocations, attributes)
    torch.cuda.synchronize()

    def probe(kinds, fn, reps):
        for k in kinds:
            mx.probe(k, a.layers * reps + 8)
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        out = {}
        for k in kinds:
            ms = mx.probe_read(k)
            mx.probe(k, 0)
            out[k] = statistics.median(ms) * 1e-3 if ms else float("nan")
        return out

    def pre():
        stack.reset()
        res.copy_(x0)
        stack.prefill_chunk(res)

    tp = probe(["in_proj", "conv", "x_proj", "dt_proj", "scan", "out_proj"], pre, 2)
    rt = torch.randn((B, D), generator=g, device="cuda")
    td = probe(["in_proj_decode", "decode_step", "out_proj"], lambda: stack.decode_step(rt), 4)
    # the persistent whole-stack decode (one cooperative launch per token over the same layers):
    # CUDA events around eager decode steps on the launching stream
    pst = MixerStack(mx, layers, B, Lp).persistent()
    res.copy_(x0)
    pst.prefill_chunk(res)
    for _ in range(3):
        pst.decode_step(rt)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        pst.decode_step(rt)
    ev[1].record()
    torch.cuda.synchronize()
    t_pst = ev[0].elapsed_time(ev[1]) / 10 * 1e-3
    K = dims.d_conv
    per_layer = (2 * E * D * 2 + D * E * 2 + P * E * 2 + E * R * 2 + E * (K + 3 + N) * 4
                 + 2 * B * E * N * 4 + 2 * B * (K - 1) * E * 2)
    ch_tok = M * E
    rows = [
        # (row, kernel, seconds, work, unit, peak, bound, work description)
        ("a1", "prefill in_proj (tcgen05)", tp["in_proj"], 2.0 * M * D * 2 * E, "flop", tc, "tensor", "2*M*D*2E"),
        ("a2", "prefill conv1d+SiLU", tp["conv"], 4.0 * ch_tok, "B", hbm, "hbm", "4 B per channel-token (x read, u write)"),
        ("a3", "prefill x_proj (tcgen05)", tp["x_proj"], 2.0 * ch_tok + 4.0 * M * P + 2.0 * P * E, "B", hbm, "hbm",
         "u read + dbc fp32 write + W_x"),
        ("a5", "prefill dt_proj+softplus (tcgen05)", tp["dt_proj"], 2.0 * M * R + 2.0 * ch_tok + 2.0 * E * R, "B", hbm,
         "hbm", "dt_low read + delta write + W_dt"),
        ("a6/a7", "prefill selective scan + gate (MUFU)", tp["scan"], 16.0 * ch_tok, "ex2", mufu, "alu",
         "16 ex2 per channel-token"),
        ("a6/a7", "prefill selective scan + gate (HBM view)", tp["scan"], 8.0 * ch_tok + 4.0 * 2 * N * M, "B", hbm,
         "hbm", "8 B per channel-token + B||C 128 B/token"),
        ("a8", "prefill out_proj (tcgen05)", tp["out_proj"], 2.0 * M * E * D, "flop", tc, "tensor", "2*M*E*D"),
        ("a10", "decode in_proj + conv step + x_proj (fused)", td["in_proj_decode"],
         2.0 * 2 * E * D + 2.0 * P * E + 2.0 * B * D + B * E * 2 * 3 + 4.0 * B * P, "B", hbm, "hbm",
         "W_in + W_x + x_in + conv window r/w + u"),
        ("a10", "decode step (AR#1 sum, dt_proj, scan step, gate)", td["decode_step"],
         2.0 * 4 * B * E * N + 2.0 * E * R + 4.0 * B * P + 2.0 * 3 * B * E, "B", hbm, "hbm",
         "h r/w fp32 + W_dt + dbc + u, z, g"),
        ("a10", "decode out_proj (split-K)", td["out_proj"], 2.0 * D * E + 2.0 * B * E + 8.0 * B * D, "B", hbm, "hbm",
         "W_out + g + residual r/w"),
        ("a10", f"persistent whole-stack decode ({a.layers} layers/launch)", t_pst,
         float(a.layers * per_layer + 2 * B * D * 4), "B", hbm, "hbm",
         "per layer W_in + W_out + W_x + W_dt + vectors + h r/w + conv window r/w; + residual"),
    ]
    out = []
    print(f"{a.config}: batch {B}, prefill M={M} tokens, d_model {D}, d_inner {E}; peaks: HBM {hbm / 1e9:.0f} GB/s, "
          f"bf16 {tc / 1e12:.0f} TF/s (burst), MUFU {mufu / 1e12:.2f} T ex2/s")
    print(f"{'row':6s} {'kernel':52s} {'us':>9s} {'achieved':>12s} {'peak':>10s} {'frac':>6s}")
    for row, name, t, work, unit, peak, bound, desc in rows:
        ach = work / t
        scale, u = {"flop": (1e12, "TFLOP/s"), "B": (1e9, "GB/s"), "ex2": (1e12, "T ex2/s")}[unit]
        print(f"{row:6s} {name:52s} {t * 1e6:9.1f} {ach / scale:9.1f} {u:>2s} {peak / scale:8.1f} {ach / peak:6.2f}")
        out.append(dict(row=row, kernel=name, us=t * 1e6, achieved=ach / scale, unit=u, peak=peak / scale,
                        frac=ach / peak, bound=bound, work=desc, work_per_launch=work))
    if a.json:
        json.dump(dict(config=a.config, batch=B, prefill_tokens=M, rows=out), open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
