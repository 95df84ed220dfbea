"""Layer stack of one TP rank: n_layers x [pre-norm RMSNorm -> TP mixer -> residual add],
chunk-major prefill carrying the per-layer SSM cache into CUDA-graph decode
(§4.1; SURVEY.md §3 call stacks (2)-(3)).  Every kernel is
launched through libssmtp's C ABI; PyTorch provides memory, streams and the graph.
"""
from __future__ import annotations

import torch

from . import _lib as L
from .mixer import LayerWeights, State, TPMixer  # noqa: F401


def synthetic_layer(dims, layer, seed=1000, device="cuda"):
    """Full (unsharded) weights of one layer generated ON the device with a seeded
    generator (same recipe as synth.layer_weights: Mamba init ranges, jittered A).
    Used for the full-depth bench where host generation of billions of parameters
    would dominate; parity tests use synth.layer_weights on the host."""
    import math
    g = torch.Generator(device=device).manual_seed(seed + layer)
    D, E, N, K, R, H = dims.d_model, dims.d_inner, dims.d_state, dims.d_conv, dims.dt_rank, dims.n_heads
    Eh = E // H
    f = dict(device=device, dtype=torch.float32)

    def u(shape, bound):
        return (torch.rand(shape, generator=g, **f) * 2 - 1) * bound

    w = {"w_in": u((2 * E, D), 1 / math.sqrt(D)), "conv_w": u((E, K), 1 / math.sqrt(K)),
         "conv_b": u((E,), 1 / math.sqrt(K)), "w_x": u((H, R + 2 * N, Eh), 1 / math.sqrt(Eh)),
         "w_dt": u((E, R), 1 / math.sqrt(R))}
    lo, hi = math.log(1e-3), math.log(1e-1)
    dt0 = torch.exp(torch.rand((E,), generator=g, **f) * (hi - lo) + lo)
    w["b_dt"] = dt0 + torch.log(-torch.expm1(-dt0))
    n = torch.arange(1, N + 1, **f)
    w["a_log"] = torch.log(n)[None, :].expand(E, N) + 0.05 * torch.randn((E, N), generator=g, **f)
    w["d_skip"] = torch.ones((E,), **f)
    w["w_out"] = u((D, E), 1 / math.sqrt(E)) / math.sqrt(2.0 * max(dims.n_layers, 1))
    return w


class DecodeStack:
    """Persistent whole-stack decode at TP = 1 (ssm_dstack_*): one cooperative launch per token runs
    every layer's pre-norm decode block (§4.1).  Owns the device buffer holding the
    re-packed projection weights and the scratch; keeps the layers' small vectors and the states'
    caches referenced (they must outlive it)."""

    def __init__(self, mixer: TPMixer, layers: list, states: list, batch: int, norm_eps=1e-5, ctas=0,
                 stream=None):
        import ctypes as C
        self.mx, self.batch = mixer, batch
        n = len(layers)
        nb = C.c_size_t()
        L.call("ssm_dstack_bytes", mixer.handle, n, batch, ctas, C.byref(nb))
        self.buf = torch.empty(nb.value, dtype=torch.uint8, device=mixer.device)
        arr = (L.ssm_layer_weights_t * n)(*[lw.struct for lw in layers])
        sts = (C.c_void_p * n)(*[st.handle.value for st in states])
        self._keep = (layers, states)
        self.handle = C.c_void_p()
        s = stream if stream is not None else torch.cuda.current_stream()
        L.call("ssm_dstack_create", mixer.handle, n, arr, sts, batch, C.c_float(norm_eps), ctas,
               C.c_void_p(self.buf.data_ptr()), nb.value, C.c_void_p(s.cuda_stream), C.byref(self.handle))

    def decode(self, res_t, stream=None):
        """res_t: [batch, D] fp32, updated in place through all layers (one kernel launch)."""
        import ctypes as C
        s = stream if stream is not None else torch.cuda.current_stream()
        L.call("ssm_dstack_decode", self.handle, C.c_void_p(res_t.data_ptr()), C.c_void_p(s.cuda_stream))

    def __del__(self):
        try:
            if self.handle:
                L.LIB.ssm_dstack_destroy(self.handle)
        except Exception:
            pass


class MixerStack:
    """flags: SSM_AR2_INT8 / SSM_AR2_FP16 / SSM_AR2_FP32 (the library's peer-to-peer AR#2), or
    SSM_AR2_EXTERNAL with nccl_group set: the NCCL bf16 all-reduce BASELINE arm (library writes the
    rank's fp32 partial, torch.distributed all-reduces it in bf16, torch adds it to the residual)."""

    def __init__(self, mixer: TPMixer, layers: list, batch: int, max_chunk: int, flags=L.SSM_AR2_INT8,
                 norm_eps=1e-5, nccl_group=None, hybrid=None):
        """hybrid: Zamba's shared transformer block as
        dict(adims=synth.AttnDims, weights={layer index: attention.SharedBlockWeights}, max_seq=int):
        before each listed layer the block runs on (residual, h0) into t, and that layer's Mamba
        block takes RMSNorm(residual + t).  The calls then take h0 (the token embeddings)."""
        self.mx, self.layers, self.batch, self.flags, self.eps = mixer, layers, batch, flags, norm_eps
        self.nccl = nccl_group if flags == L.SSM_AR2_EXTERNAL else None
        d = mixer.dims
        dt = torch.bfloat16 if mixer.dtype == "bf16" else torch.float32
        self.ws = mixer.workspace(batch, max_chunk, flags)
        self.ws_dec = mixer.workspace(batch, 1, flags)
        self.xbuf = torch.empty((batch * max_chunk, d.d_model), dtype=dt, device=mixer.device)
        self.xbuf_dec = torch.empty((batch, d.d_model), dtype=dt, device=mixer.device)
        self.states = [State(mixer, batch) for _ in layers]
        if self.nccl is not None:
            self.part = torch.empty((batch * max_chunk, d.d_model), dtype=torch.float32, device=mixer.device)
        self.hybrid = {}
        if hybrid:
            from .attention import SharedBlock
            shared_ws = None
            for li, w in hybrid["weights"].items():
                blk = SharedBlock(mixer, hybrid["adims"], batch, hybrid["max_seq"], max_chunk, workspaces=shared_ws)
                shared_ws = (blk.ws, blk.ws_dec)      # one workspace pair for every hybrid layer
                self.hybrid[li] = (w, blk)
            self.t_buf = torch.empty((batch * max_chunk, d.d_model), device=mixer.device)
            self.h0_dec = torch.zeros((batch, d.d_model), device=mixer.device)
        # prefill with the pre-norm folded around the projections (ssm_mixer_prefill_normed): x =
        # bf16(residual) and its row statistic come from the kernel that finished the previous layer's
        # residual rows -- the out_proj epilogue at TP = 1, the int8 AR#2's reduce / all-gather at TP > 1
        other_ar2 = L.SSM_AR2_FP16 | L.SSM_AR2_BF16 | L.SSM_AR2_FP32 | L.SSM_AR2_EXTERNAL | L.SSM_QAR_REQUANT
        self.prefill_normed = (mixer.dtype == "bf16" and not self.hybrid and self.nccl is None
                               and not (flags & L.SSM_TP_NAIVE)
                               and (mixer.tp_size == 1 or (not (flags & other_ar2) and d.d_model % 32 == 0)))
        if self.prefill_normed:
            self.ssbuf = torch.empty((2, (batch * max_chunk + 3) // 4 * 4), dtype=torch.float32, device=mixer.device)
        self.graph = None
        self.graph_launches = 0
        self._graph_parity = 0
        self.dec_flags = 0   # extra decode flags (SSM_DECODE_UNFUSED: cross-checks)
        self.dstack = None   # DecodeStack: the persistent whole-stack decode (TP = 1), see persistent()

    def persistent(self, ctas=0):
        """Switch decode to the persistent whole-stack kernel (TP = 1, pure Mamba stacks); raises
        SSMError(SSM_ERR_UNSUPPORTED) for shapes it does not cover."""
        if self.hybrid or self.nccl is not None:
            raise ValueError("persistent decode: pure Mamba stacks without the NCCL arm only")
        self.dstack = DecodeStack(self.mx, self.layers, self.states, self.batch, self.eps, ctas)
        return self

    def reset(self, stream=None):
        for s in self.states:
            s.reset(stream)
        for _, blk in self.hybrid.values():
            blk.reset(stream)

    def prefill_chunk(self, res, stream=None, h0=None):
        """res: [batch * Lc, D] fp32, this chunk's residual rows (row = b*Lc + t), updated in place;
        h0: the chunk's token embeddings (Zamba hybrid layers)."""
        n = res.shape[0]
        x = self.xbuf[:n]
        if self.prefill_normed:
            ss = self.ssbuf[:, :n]
            self.mx.rowstats(res, x, ss[0], stream)
            last = len(self.layers) - 1
            for li, (lw, st) in enumerate(zip(self.layers, self.states)):
                nxt = li < last
                self.mx.prefill_normed(lw, st, x, ss[li & 1], res, x if nxt else None, ss[(li + 1) & 1] if nxt else None,
                                       self.eps, self.flags, self.ws, stream)
            return
        for li, (lw, st) in enumerate(zip(self.layers, self.states)):
            if li in self.hybrid:
                w, blk = self.hybrid[li]
                t = self.t_buf[:n]
                blk(w, res, h0, t, n // self.batch, self.flags & (L.SSM_AR2_INT8 | L.SSM_AR2_FP16 | L.SSM_AR2_BF16),
                    stream)
                self.mx.rmsnorm_add(res, t, x, None, self.eps, stream)
            else:
                self.mx.rmsnorm(res, x, None, self.eps, stream)
            if self.nccl is None:
                self.mx.prefill(lw, st, x, res, self.flags, self.ws, stream)
            else:
                self._nccl_layer(lambda p: self.mx.prefill(lw, st, x, p, self.flags, self.ws, stream), res)

    def decode_step(self, res_t, stream=None):
        """res_t: [batch, D] fp32, updated in place through all layers (ssm_mixer_decode_block:
        pre-norm RMSNorm, then the layer's decode kernels); Zamba hybrid layers read the token
        embeddings from self.h0_dec."""
        if self.dstack is not None:
            self.dstack.decode(res_t, stream)
            return
        for li, (lw, st) in enumerate(zip(self.layers, self.states)):
            if li in self.hybrid:
                w, blk = self.hybrid[li]
                t = self.t_buf[:self.batch]
                blk(w, res_t, self.h0_dec, t, 1, self.flags & (L.SSM_AR2_INT8 | L.SSM_AR2_FP16 | L.SSM_AR2_BF16),
                    stream)
                self.mx.rmsnorm_add(res_t, t, self.xbuf_dec, None, self.eps, stream)
                if self.nccl is None:
                    self.mx.decode(lw, st, self.xbuf_dec, res_t, self.flags | self.dec_flags, self.ws_dec, stream)
                else:
                    self._nccl_layer(lambda p: self.mx.decode(lw, st, self.xbuf_dec, p, self.flags, self.ws_dec,
                                                              stream), res_t)
                continue
            if self.nccl is None:
                self.mx.decode_block(lw, st, res_t, self.eps, self.flags | self.dec_flags, self.ws_dec, stream)
            else:
                self.mx.rmsnorm(res_t, self.xbuf_dec, None, self.eps, stream)
                self._nccl_layer(lambda p: self.mx.decode(lw, st, self.xbuf_dec, p, self.flags, self.ws_dec, stream),
                                 res_t)

    def _nccl_layer(self, run, res):
        import torch.distributed as dist
        p = self.part[:res.shape[0]]
        run(p)                                   # p := this rank's fp32 partial out_proj
        pb = p.to(torch.bfloat16)
        dist.all_reduce(pb, group=self.nccl)     # NCCL bf16 all-reduce (baseline arm)
        res.add_(pb.float())

    def capture_decode(self, res_t, probes=(), warmup=True):
        """Capture one decode step over all layers into a CUDA graph reading/writing res_t.
        The decode path is graph-safe: no host sync, fixed pointers; the all-reduce epoch
        counters live in device memory and advance on every replay.  The symmetric-buffer halves
        of the captured collectives are fixed, so the graph must be replayed with the handle's
        epoch at the parity it had at capture (replay() realigns it with a barrier), and one step
        must issue an even number of collectives so that back-to-back replays alternate halves."""
        if warmup:  # one eager step first (attribute setup outside capture); callers driving several
            s = torch.cuda.Stream()  # virtual ranks on one device do their warm-ups themselves
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.decode_step(res_t, s)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
        for kind, cap in probes:  # event nodes recorded inside the graph (see SSM_PROBE_IN_PROJ_DECODE)
            self.mx.probe(kind, cap)
        g = torch.cuda.CUDAGraph()
        before = self.mx.launches()
        ar_before = self.mx.stats()["allreduce"]
        self._graph_parity = self.mx.epoch() & 1
        e0 = self.mx.epoch()
        with torch.cuda.graph(g):
            self.decode_step(res_t)
            if (self.mx.epoch() - e0) % 2:  # odd collective count (e.g. Zamba at TP = 2): one payload-free
                self.mx.barrier()              # barrier keeps back-to-back replays alternating the halves
        self.graph_launches = self.mx.launches() - before
        if (self.mx.epoch() - e0) % 2:
            raise RuntimeError("odd number of collectives per decode step: double-buffer halves would not alternate")
        del ar_before
        self.graph = g
        return g

    def align_epoch(self, stream=None):
        """Before replaying the decode graph: if eager collectives since the capture (a prefill)
        left the epoch at the other parity, one payload-free barrier restores it."""
        if self.mx.tp_size > 1 and (self.mx.epoch() & 1) != self._graph_parity:
            self.mx.barrier(stream)

    def replay(self, graph=None, stream=None):
        self.align_epoch(stream)
        (graph or self.graph).replay()
