#!/usr/bin/env python
"""Per-CTA timeline of one decode-GEMM launch (experiment tool, GPU only).  Runs the swap-AB
packed GEMM under CUDA-graph replay with SSM_GEMM_NOMMA bit 8 (trace) plus optional experiment
bits from argv, then prints each pipeline event's clock64 offset from CTA entry (us at the
SM clock) over the CTAs of the last launch, and the globaltimer spread of CTA entry/exit.
    SSM_GEMM_NOMMA=8 python scripts/gemm_trace.py [M N K]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import TPMixer, _lib as L  # noqa: E402

NAMES = ["gt_entry", "clk_entry", "prologue_done", "tma_first_issue", "mma_first_full", "mma_last_full",
         "mma_done_commit", "epi_tfull", "epi_tmem_ld", "epi_stores_done", "cta_end_sync", "dealloc_done",
         "gt_exit"]


def main():
    M, N, K = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (16, 10240, 2560)
    mx = TPMixer(synth.CONFIGS["tiny"], "bf16")
    copies = 8
    W = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(copies)]
    PK = [mx.pack_weight(w) for w in W]
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda")
    for i in range(2):
        mx.dbg_gemm_packed(X, W[i], PK[i], C)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    reps = 24
    with torch.cuda.graph(g):
        for i in range(reps):
            mx.dbg_gemm_packed(X, W[i % copies], PK[i % copies], C)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    ctas = min(148, (N + 127) // 128)
    buf = (ctypes.c_uint64 * (1024 * 16))()
    L.call("ssm_dbg_gemm_trace", buf, 1024 * 16)
    t = np.array(buf[:ctas * 16], dtype=np.float64).reshape(ctas, 16)
    ghz = 1.965
    print(f"M={M} N={N} K={K} NOMMA={os.environ.get('SSM_GEMM_NOMMA')}: {us:.2f} us/launch (graph), {ctas} CTAs")
    for j in range(2, 12):
        v = t[:, j] / ghz / 1000
        print(f"  {NAMES[j]:16s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
    ge = (t[:, 0] - t[:, 0].min()) / 1000
    gx = (t[:, 12] - t[:, 0].min()) / 1000
    print(f"  entry spread (globaltimer) {ge.max():.2f} us; exit min {gx.min():.2f} med {np.median(gx):.2f} "
          f"max {gx.max():.2f} us after first entry")


if __name__ == "__main__":
    main()
