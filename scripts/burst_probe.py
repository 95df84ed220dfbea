"""Do TMA bulk copies of one SM overlap, and what does it cost when all SMs read the SAME bytes?
Each CTA issues n copies of ch bytes at once and waits (scripts/stream_probe.cu bulk_burst)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from stream_probe import build  # noqa: E402

lib = build()
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
buf = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
buf.fill_(1)


def t(grid, n, ch, span, reps=20, issuers=1, rewrite=False):
    f = lambda: lib.probe_burst(ctypes.c_void_p(buf.data_ptr()), ctypes.c_longlong(span), grid, n, ch, reps,
                                issuers, ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(st))
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if rewrite:
        buf[:span].add_(1)  # freshly written (dirty) lines
    e0.record()
    f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps


for n, ch in ((22, 2048), (11, 2048), (8, 16384)):
    for span_name, span in (("distinct", buf.numel()), ("shared-80KB", 80 * 1024 + n * ch), ("same", n * ch + 16)):
        us = t(148, n, ch, span, issuers=32)
        print(f"grid 148 n={n:2d} ch={ch:5d} {span_name:12s}: {us:7.2f} us per burst ({148 * n * ch / us / 1e3:7.0f} GB/s total)",
              flush=True)
