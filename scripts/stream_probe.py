#!/usr/bin/env python
"""Single-launch HBM read-rate probe for decode-sized weight streams (GPU only, experiment tool).
Compiles scripts/stream_probe.cu, then times (CUDA-graph replay, buffers rotating beyond L2)
one launch reading B bytes with LDG.128 or a cp.async.bulk ring, across grid sizes.
    python scripts/stream_probe.py
"""
import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "..", "build", "stream_probe.so")


def build():
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "stream_probe.cu")])
    return ctypes.CDLL(SO)


def timeit(fn, bufs, reps=24):
    for i in range(2):
        fn(bufs[i % len(bufs)])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(bufs[i % len(bufs)])
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps


def main():
    lib = build()
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    for mb in (52.4288, 26.2144, 6.5536):
        nbytes = int(mb * 1e6) // 4096 * 4096
        copies = max(2, int(400e6 // nbytes))
        bufs = [torch.empty(nbytes, dtype=torch.uint8, device="cuda").fill_(i) for i in range(copies)]

        def run(label, fn):
            us = timeit(fn, bufs)
            print(f"{mb:7.2f} MB {label:34s}: {us:7.2f} us  {nbytes / us / 1e3:7.1f} GB/s", flush=True)

        for grid, block in ((148, 512), (296, 512), (592, 256), (1184, 256), (80, 512)):
            run(f"ldg grid={grid} block={block}",
                lambda b: lib.probe_ldg(ctypes.c_void_p(b.data_ptr()), ctypes.c_longlong(nbytes), grid, block,
                                        ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) or None)
        for grid, S, CH in ((148, 8, 16384), (148, 12, 16384), (148, 6, 32768), (80, 12, 16384), (80, 6, 32768),
                            (296, 6, 16384), (148, 24, 8192)):
            run(f"bulk grid={grid} S={S} CH={CH}",
                lambda b: lib.probe_bulk(ctypes.c_void_p(b.data_ptr()), ctypes.c_longlong(nbytes), grid, S, CH,
                                         ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) or None)
        del bufs


if __name__ == "__main__":
    main()
