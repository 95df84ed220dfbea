#!/usr/bin/env python
"""Microbenchmark of the prefill scan kernel on Mamba-2.8B shapes (GPU only).
    python scripts/scan_micro.py [--tp 1] [--batch 16] [--seqlen 2048]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import TPMixer  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--tp", type=int, default=1)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--seqlen", type=int, default=2048)
    a = p.parse_args()
    dims = synth.CONFIGS["mamba2.8b"]
    mx = TPMixer(dims, "bf16", rank=0, tp_size=1) if a.tp == 1 else None
    if mx is None:  # emulate the rank-local channel count of TP=k with a TP=1 handle of E/k channels
        d = synth.MixerDims(d_model=dims.d_model // a.tp, d_inner=dims.d_inner // a.tp, dt_rank=dims.dt_rank)
        mx = TPMixer(d, "bf16")
    E, N, B, L = mx.ek, 16, a.batch, a.seqlen
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(B * L, E, device="cuda", generator=g).to(torch.bfloat16)
    dl = (torch.rand(B * L, E, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    z = torch.randn(B * L, E, device="cuda", generator=g).to(torch.bfloat16)
    BC = torch.randn(B * L, 2 * N, device="cuda", generator=g)
    a_log = torch.log(torch.arange(1, N + 1, device="cuda").float())[None].expand(E, N).contiguous()
    dsk = torch.ones(E, device="cuda")
    h = torch.zeros(B, E, N, device="cuda")
    out = torch.empty(B * L, E, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        mx.dbg_scan(u, dl, z, E, BC, a_log, dsk, h, out, B, L)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        mx.dbg_scan(u, dl, z, E, BC, a_log, dsk, h, out, B, L)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    chtok = B * L * E
    byts = chtok * 8 + B * L * 2 * N * 4
    print(f"scan tp={a.tp} B={B} L={L} E_k={E}: {ms * 1000:8.1f} us  "
          f"{chtok / ms / 1e6:8.1f} Gch-tok/s  {byts / ms / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
