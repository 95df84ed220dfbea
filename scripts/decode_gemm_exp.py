#!/usr/bin/env python
"""Controlled experiments on the decode (swap-AB, weight-streaming) GEMM: device time per call
under CUDA-graph replay, weights rotating beyond L2, for library env knobs
(SSM_GEMM_KBS, SSM_GEMM_NOMMA, SSM_GEMM_RING_KB, SSM_GEMM_SK_CTAS).  GPU only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200 import TPMixer  # noqa: E402

EXPS = [
    ("packed nomma|noB", {"PACK": "1", "SSM_GEMM_NOMMA": "3"}, 1),
    ("packed nomma|noB|noepi", {"PACK": "1", "SSM_GEMM_NOMMA": "7"}, 1),
    ("packed noB", {"PACK": "1", "SSM_GEMM_NOMMA": "2"}, 1),
    ("packed nomma", {"PACK": "1", "SSM_GEMM_NOMMA": "1"}, 1),
    ("packed kbs2", {"PACK": "1"}, 1),
    ("packed kbs1", {"PACK": "1", "SSM_GEMM_KBS": "1"}, 1),
    ("packed kbs4", {"PACK": "1", "SSM_GEMM_KBS": "4"}, 1),
    ("packed split2", {"PACK": "1"}, 2),
    ("packed streamK148", {"PACK": "1"}, -1),
    ("base kbs2", {}, 1),
    ("kbs1", {"SSM_GEMM_KBS": "1"}, 1),
    ("nomma", {"SSM_GEMM_NOMMA": "1"}, 1),
    ("streamK148", {}, -1),
]
SHAPES = {"in_proj": (16, 10240, 2560), "in_proj_K1280": (16, 10240, 1280), "in_proj_K640": (16, 10240, 640),
          "out_proj": (16, 2560, 5120)}


def main():
    mx = TPMixer(synth.CONFIGS["tiny"], "bf16")
    keys = {k for _, e, _ in EXPS for k in e}
    for sname, (M, N, K) in SHAPES.items():
        copies = 8
        X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda")
        # cuBLAS reference on the same shape (library GEMM, for calibration only)
        Wc = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(copies)]
        for i in range(3):
            torch.matmul(X, Wc[i].T)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(24):
            torch.matmul(X, Wc[i % copies].T)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / 24
        print(f"{sname:9s} {'cuBLAS torch.matmul (eager)':28s}      : {us:8.2f} us  {N * K * 2 / (us * 1e-6) / 1e9:8.1f} GB/s",
              flush=True)
        del Wc
        for name, env, ks in EXPS:
            pad = int(env.get("PAD", "0"))
            Wfull = [torch.randn(N, K + pad, device="cuda").to(torch.bfloat16) for _ in range(copies)]
            W = [w[:, :K] for w in Wfull]
            for k in keys:
                os.environ.pop(k, None)
            os.environ.update({k: v for k, v in env.items() if k not in ("PAD", "PACK")})
            packed = env.get("PACK") == "1"
            PK = [mx.pack_weight(w.contiguous()) for w in W] if packed else None
            torch.cuda.synchronize()

            def call(i):
                if packed:
                    mx.dbg_gemm_packed(X, W[i], PK[i], C, ksplit=ks)
                else:
                    mx.dbg_gemm_ld(X, W[i], C, M, N, K, swap_ab=True, ksplit=ks)
            reps = 24
            for i in range(2):
                call(i)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(reps):
                    call(i % copies)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1000 / reps
            print(f"{sname:9s} {name:28s} ks={ks:2d}: {us:8.2f} us  {N * K * 2 / (us * 1e-6) / 1e9:8.1f} GB/s"
                  f"{'  (incl memset)' if ks != 1 else ''}", flush=True)
            del g, W, Wfull, PK


if __name__ == "__main__":
    main()
