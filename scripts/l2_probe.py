"""Bulk-copy ring read rate from HBM vs L2-resident data (experiment tool).
Uses scripts/stream_probe.cu's bulk_stream kernel."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from stream_probe import build  # noqa: E402

lib = build()
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def run(buf, nbytes, S=8, CH=16384, grid=148):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.probe_bulk(ctypes.c_void_p(buf.data_ptr()), ctypes.c_longlong(nbytes), grid, S, CH,
                   ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(s))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000


big = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")  # 4 GB: rotate to defeat L2
for nb in (26 << 20, 52 << 20):
    for S in (4, 8, 12):
        # cold: a fresh region each time
        cold = []
        for r in range(6):
            off = (r * 97 + 13) * (64 << 20) % ((4 << 30) - nb)
            cold.append(run(big[off:], nb, S))
        # warm: same region read twice back to back (second read L2-resident, 52 MB < L2)
        warm = []
        for r in range(6):
            run(big, nb, S)
            warm.append(run(big, nb, S))
        print(f"{nb/1e6:6.1f} MB S={S:2d}: cold {min(cold):7.2f} us ({nb/min(cold)/1e3:6.0f} GB/s)   "
              f"L2-warm {min(warm):7.2f} us ({nb/min(warm)/1e3:6.0f} GB/s)", flush=True)
