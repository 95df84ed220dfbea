"""Layer stack of one TP rank: n_layers x [pre-norm RMSNorm -> TP mixer -> residual add],
chunk-major prefill carrying the per-layer SSM cache into CUDA-graph decode
(§4.1; SURVEY.md §3 call stacks (2)-(3)).  Every kernel is
launched through libssmtp's C ABI; PyTorch provides memory, streams and the graph.
"""
from __future__ import annotations

import os

from ctypes import c_float as C_float

import torch

from . import _lib as L

_DEBUG_SKIP_NORM = os.environ.get("SSM_DEBUG_SKIP_NORM") == "1"  # timing ablations only
from .mixer import LayerWeights, State, TPMixer


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


class MixerStack:
    """flags: SSM_AR2_INT8 / SSM_AR2_FP32 (the library's peer-to-peer AR#2), or SSM_AR2_EXTERNAL
    with nccl_group set: the NCCL bf16 all-reduce BASELINE arm (library writes the rank's fp32
    partial, torch.distributed all-reduces it in bf16, torch adds it to the residual)."""

    def __init__(self, mixer: TPMixer, layers: list, batch: int, max_chunk: int, flags=L.SSM_AR2_INT8,
                 norm_eps=1e-5, nccl_group=None, persistent=None):
        """persistent: decode every token with ONE launch of the persistent whole-stack kernel
        (ssm_stack_decode) when the library supports the configuration (TP=1, bf16, packed
        weights, ...).  True = required; False = per-layer calls; None = the environment's
        SSM_PERSISTENT_DECODE=1 opts in (default off: measured slower than the per-layer graph,
        DESIGN.md §6c)."""
        self.mx, self.layers, self.batch, self.flags, self.eps = mixer, layers, batch, flags, norm_eps
        self.nccl = nccl_group if flags == L.SSM_AR2_EXTERNAL else None
        d = mixer.dims
        dt = torch.bfloat16 if mixer.dtype == "bf16" else torch.float32
        self.ws = mixer.workspace(batch, max_chunk)
        self.ws_dec = mixer.workspace(batch, 1)
        self.xbuf = torch.empty((batch * max_chunk, d.d_model), dtype=dt, device=mixer.device)
        self.xbuf_dec = torch.empty((batch, d.d_model), dtype=dt, device=mixer.device)
        self.states = [State(mixer, batch) for _ in layers]
        if self.nccl is not None:
            self.part = torch.empty((batch * max_chunk, d.d_model), dtype=torch.float32, device=mixer.device)
        self.graph = None
        self.graph_launches = 0
        self.stack_ws = None
        # opt-in (SSM_PRENORM=1): the pre-norm computed inside the fused decode in_proj
        # (ssm_mixer_decode_prenorm).  Measured slower: 44.6 vs 38.0 us per Mamba-2.8B decode layer
        # -- 80 CTAs re-reading the same 164 KB of residual rows from L2 cost more than the 16-block
        # norm kernel they replace
        self.prenorm = mixer.dtype == "bf16" and os.environ.get("SSM_PRENORM", "0") == "1"
        self.chain = False  # per-layer decode with the pre-norm folded into the GEMMs (ssm_mixer_decode_chained)
        # opt-in (SSM_DECODE_CHAIN=1): measured slower than the norm kernel it removes
        if self.nccl is None and os.environ.get("SSM_DECODE_CHAIN", "0") == "1" and layers:
            import ctypes as C
            ok = C.c_int32(0)
            L.call("ssm_decode_chain_supported", mixer.handle, C.byref(layers[0].struct), batch, C.byref(ok))
            self.chain = bool(ok.value)
        required = bool(persistent)
        if persistent is None:
            persistent = os.environ.get("SSM_PERSISTENT_DECODE") == "1"
        if persistent and self.nccl is None:
            self._bind_persistent(required=required)

    def _bind_persistent(self, required=False):
        import ctypes as C
        from .mixer import _ptr, _stream
        nl = len(self.layers)
        nb = C.c_size_t()
        rc = L.LIB.ssm_stack_bytes(self.mx.handle, nl, self.batch, C.byref(nb))
        packed = all(lw.struct.w_in_pk and lw.struct.w_out_pk for lw in self.layers)
        if rc != 0 or not packed:
            if required:
                raise L.SSMError(rc or 8, "ssm_stack_bytes", L.LIB.ssm_last_error().decode() if rc else
                                 "layers are not packed (LayerWeights.pack)")
            return
        self._layer_arr = (L.ssm_layer_weights_t * nl)(*[lw.struct for lw in self.layers])
        self._state_arr = (C.c_void_p * nl)(*[st.handle.value for st in self.states])
        self.stack_ws = torch.zeros(nb.value, dtype=torch.uint8, device=self.mx.device)
        L.call("ssm_stack_bind", self.mx.handle, C.cast(self._layer_arr, C.c_void_p), C.cast(self._state_arr, C.c_void_p), nl, self.batch,
               _ptr(self.stack_ws), nb.value, _stream(None))

    def stack_check(self, stream=None):
        from .mixer import _ptr, _stream
        if self.stack_ws is not None:
            L.call("ssm_stack_check", self.mx.handle, _ptr(self.stack_ws), _stream(stream))

    def reset(self, stream=None):
        for s in self.states:
            s.reset(stream)

    def prefill_chunk(self, res, stream=None):
        """res: [batch * Lc, D] fp32, this chunk's residual rows (row = b*Lc + t), updated in place."""
        n = res.shape[0]
        x = self.xbuf[:n]
        for lw, st in zip(self.layers, self.states):
            self.mx.rmsnorm(res, x, None, self.eps, stream)
            if self.nccl is None:
                self.mx.prefill(lw, st, x, res, self.flags, self.ws, stream)
            else:
                self._nccl_layer(lambda p: self.mx.prefill(lw, st, x, p, self.flags, self.ws, stream), res)

    def decode_step(self, res_t, stream=None):
        """res_t: [batch, D] fp32, updated in place through all layers."""
        if self.stack_ws is not None:
            from .mixer import _ptr, _stream
            L.call("ssm_stack_decode", self.mx.handle, _ptr(self.stack_ws), _ptr(res_t), C_float(self.eps),
                   _stream(stream))
            return
        if self.chain:
            import ctypes as C
            from .mixer import _ptr, _stream
            L.call("ssm_decode_chain_begin", self.mx.handle, _ptr(res_t), _ptr(self.xbuf_dec), self.batch,
                   _ptr(self.ws_dec), self.ws_dec.numel(), _stream(stream))
            for lw, st in zip(self.layers, self.states):
                L.call("ssm_mixer_decode_chained", self.mx.handle, C.byref(lw.struct), st.handle, _ptr(self.xbuf_dec),
                       _ptr(res_t), self.batch, C.c_float(self.eps), _ptr(self.ws_dec), self.ws_dec.numel(),
                       _stream(stream))
            return
        if self.prenorm and self.nccl is None and not _DEBUG_SKIP_NORM:
            import ctypes as C
            from .mixer import _ptr, _stream
            for lw, st in zip(self.layers, self.states):
                L.call("ssm_mixer_decode_prenorm", self.mx.handle, C.byref(lw.struct), st.handle, _ptr(self.xbuf_dec),
                       _ptr(res_t), self.batch, C.c_float(self.eps), self.flags, _ptr(self.ws_dec),
                       self.ws_dec.numel(), _stream(stream))
            return
        skip_norm = _DEBUG_SKIP_NORM
        for lw, st in zip(self.layers, self.states):
            if not skip_norm:
                self.mx.rmsnorm(res_t, self.xbuf_dec, None, self.eps, stream)
            if self.nccl is None:
                self.mx.decode(lw, st, self.xbuf_dec, res_t, self.flags, self.ws_dec, stream)
            else:
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
        counters live in device memory and advance on every replay, and each step issues an
        even number of collectives so the double-buffer halves alternate across replays."""
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
        with torch.cuda.graph(g):
            self.decode_step(res_t)
        self.graph_launches = self.mx.launches() - before
        if (self.mx.stats()["allreduce"] - ar_before) % 2:
            raise RuntimeError("odd number of collectives per decode step: double-buffer halves would not alternate")
        self.graph = g
        return g
