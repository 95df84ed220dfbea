"""Cost of mbarrier.try_wait / test_wait on a completed phase and of reading %globaltimer (cycles)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from stream_probe import build  # noqa: E402

lib = build()
out = torch.zeros(4, dtype=torch.int64, device="cuda")
lib.probe_mbar(ctypes.c_void_p(out.data_ptr()), 1000, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("cycles per call: try_wait(complete) %d, test_wait(complete) %d, globaltimer read %d (ok count %d)" % tuple(out.tolist()))
