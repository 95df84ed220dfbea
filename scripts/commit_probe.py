"""Cycles to probe 22 completed mbarriers arrived by threads (mode 0) vs by tcgen05.commit (mode 1)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from stream_probe import build  # noqa: E402

lib = build()
out = torch.zeros(8, dtype=torch.int64, device="cuda")
lib.probe_commit(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
o = out.tolist()
print(f"thread-arrived: 22 probes {o[0]} cyc (again {o[1]}), ok={o[2]}; tcgen05.commit-arrived: {o[4]} cyc (again {o[5]}), ok={o[6]}")
