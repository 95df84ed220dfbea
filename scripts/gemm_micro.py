#!/usr/bin/env python
"""Microbenchmark of the tcgen05 GEMM on the mixer's projection shapes (GPU only).

Calls are captured into a CUDA graph (decode-sized GEMMs are otherwise host-launch bound),
and weights rotate over enough copies to exceed L2 (126 MB) so weight-streaming decode GEMMs
read HBM as in a real decode step.  Prints device time per call, TFLOP/s and GB/s.
    python scripts/gemm_micro.py [--only dec] [--kbs 1,2]
"contig" rows reproduce the decode in_proj byte count with K=64, so every 128-row TMA box is
one contiguous 16 KB block (a DRAM-locality experiment, not a mixer shape).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import TPMixer, _lib as L  # noqa: E402

SHAPES = {
    # name: (tokens M, out features N, K, swap_ab, ksplit)
    "dec_in_proj": (16, 10240, 2560, 1, 1),
    "dec_in_proj_sk": (16, 10240, 2560, 1, -1),
    "dec_in_proj_contig": (16, 10240 * 40, 64, 1, 1),
    "dec_x_proj": (16, 192, 5120, 1, 32),
    "dec_x_proj_sk": (16, 192, 5120, 1, -1),
    "dec_out_proj": (16, 2560, 5120, 1, 7),
    "dec_out_proj_sk": (16, 2560, 5120, 1, -1),
    "dec_out_proj_contig": (16, 2560 * 80, 64, 1, 1),
    "pre_in_proj": (32768, 10240, 2560, 0, 1),
    "pre_x_proj": (32768, 192, 5120, 0, 1),
    "pre_dt_proj": (32768, 5120, 160, 0, 1),
    "pre_out_proj": (32768, 2560, 5120, 0, 1),
}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--only", default="")
    p.add_argument("--pair", default="-1", help="CTA-pair GEMM modes to time (ssm_dbg_set_gemm_pair), e.g. 0,1")
    a = p.parse_args()
    for mode in [int(v) for v in a.pair.split(",")]:
        L.call("ssm_dbg_set_gemm_pair", mode)
        print(f"-- gemm pair mode {mode}", flush=True)
        run(a)
    L.call("ssm_dbg_set_gemm_pair", -1)


def run(a):
    mx = TPMixer(synth.CONFIGS["tiny"], "bf16")
    for name, (M, N, K, swap, ks) in SHAPES.items():
        if a.only and a.only not in name:
            continue
        wbytes = N * K * 2
        copies = max(1, min(8, int(3 * 126e6 // wbytes) + 1)) if swap else 1
        W = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(copies)]
        X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda")
        for kbs in ("auto",):
            reps = 24 if swap else 4
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for i in range(2):
                    mx.dbg_gemm(X, W[i % copies], C, swap_ab=bool(swap), ksplit=ks, stream=s)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(reps):
                    mx.dbg_gemm(X, W[i % copies], C, swap_ab=bool(swap), ksplit=ks)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1000 / reps
            tf = 2 * M * N * K / (us * 1e-6) / 1e12
            gbs = (wbytes + M * K * 2 + M * N * 4) / (us * 1e-6) / 1e9
            extra = " (incl. memset)" if ks != 1 else ""
            print(f"{name:20s} M={M:6d} N={N:7d} K={K:5d} swap={swap} ks={ks:2d} kbs={kbs}: "
                  f"{us:9.2f} us  {tf:8.1f} TFLOP/s  {gbs:8.1f} GB/s{extra}", flush=True)
            del g


if __name__ == "__main__":
    main()
