"""k virtual TP ranks on ONE GPU (SSM_COMM_VIRTUAL): same-device symmetric buffers and one CUDA
stream per rank, so the real peer-to-peer all-reduce kernels and their flag protocol run without
a second GPU.  Used by the -m gpu tests and by the agreement harness (generate.py)."""
from __future__ import annotations

import torch

from . import _lib as L
from .mixer import TPMixer


class VirtualGroup:
    def __init__(self, dims, k, dtype, max_tokens, qar_block=128):
        self.k = k
        cfg = L.make_config(dims, dtype, qar_block)
        nbytes = L.comm_bytes(cfg, k, max_tokens)
        self.bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(k)]
        ptrs = [b.data_ptr() for b in self.bufs]
        self.mixers = [TPMixer(dims, dtype, rank=r, tp_size=k, peer_bufs=ptrs, buf_bytes=nbytes, virtual=True,
                               qar_block=qar_block) for r in range(k)]
        self.streams = [torch.cuda.Stream() for _ in range(k)]
        torch.cuda.synchronize()

    def run(self, fn):
        """fn(rank, mixer, stream) enqueues rank r's work on its own stream; returns after all ranks
        finished and their device error words were checked."""
        ev = torch.cuda.Event()
        ev.record()
        for r in range(self.k):
            self.streams[r].wait_event(ev)
        for r in range(self.k):
            with torch.cuda.stream(self.streams[r]):
                fn(r, self.mixers[r], self.streams[r])
        for s in self.streams:
            torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        for r in range(self.k):
            self.mixers[r].check(self.streams[r])
