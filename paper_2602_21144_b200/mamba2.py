"""Mamba-2 (SSD) mixer on one TP rank: Python
marshalling over ssm_m2_* (include/ssm_tp.h).  The rank's slices of the packed parameters
(reading M1): rows z_r | x_r | B | C | dt_r of W_in (B, C replicated: n_groups == 1), the conv taps
of its x channels then of B, C, its heads' dt_bias / A_log / D, its norm-weight entries and
W_out columns."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from .mixer import _ptr, _stream


def m2_config(m2):
    return L.ssm_m2_config_t(m2.d_inner, m2.d_state, m2.headdim, m2.n_groups, m2.d_conv, m2.eps)


class Mamba2Weights:
    def __init__(self, m2, full, tp_size=1, rank=0, device="cuda"):
        E, N, G, H = m2.d_inner, m2.d_state, m2.n_groups, m2.n_heads
        Ek, Hk = E // tp_size, H // tp_size
        ch = torch.arange(rank * Ek, (rank + 1) * Ek)
        hs = torch.arange(rank * Hk, (rank + 1) * Hk)
        bc = torch.arange(2 * G * N)
        conv_dim = E + 2 * G * N
        rows = torch.cat([ch, E + ch, 2 * E + bc, E + conv_dim + hs])
        cidx = torch.cat([ch, E + bc])

        def bf(t):
            return t.to(device=device, dtype=torch.bfloat16).contiguous()

        def f32(t):
            return t.to(device=device, dtype=torch.float32).contiguous()

        self.tensors = {"w_in": bf(full["w_in"][rows]), "conv_w": f32(full["conv_w"][cidx]),
                        "conv_b": f32(full["conv_b"][cidx]), "dt_bias": f32(full["dt_bias"][hs]),
                        "a_log": f32(full["a_log"][hs]), "d_skip": f32(full["d_skip"][hs]),
                        "norm_w": f32(full["norm_w"][ch]), "w_out": bf(full["w_out"][:, ch])}
        self.struct = L.ssm_m2_weights_t(**{k: v.data_ptr() for k, v in self.tensors.items()})


class Mamba2Mixer:
    """One layer's cache + calls on this rank of `mixer` (a TPMixer supplying d_model and the
    communicator)."""

    def __init__(self, mixer, m2, batch, max_chunk, stream=None):
        self.mx, self.m2, self.batch = mixer, m2, batch
        self.cfg = m2_config(m2)
        cb, hb = C.c_size_t(), C.c_size_t()
        L.call("ssm_m2_state_bytes", mixer.handle, C.byref(self.cfg), batch, C.byref(cb), C.byref(hb))
        self.conv = torch.zeros(cb.value // 2, dtype=torch.bfloat16, device=mixer.device)
        self.h = torch.zeros(hb.value // 4, dtype=torch.float32, device=mixer.device)
        self.ws = self.workspace(max_chunk)
        self.ws_dec = self.workspace(1)

    def workspace(self, seqlen):
        nb = C.c_size_t()
        L.call("ssm_m2_workspace_bytes", self.mx.handle, C.byref(self.cfg), self.batch, seqlen, C.byref(nb))
        return torch.empty(max(nb.value, 256), dtype=torch.uint8, device=self.mx.device)

    def reset(self):
        self.conv.zero_()
        self.h.zero_()

    def __call__(self, w, x_in, residual, seqlen, flags=L.SSM_AR2_INT8, stream=None):
        ws = self.ws_dec if seqlen == 1 else self.ws
        L.call("ssm_m2_mixer", self.mx.handle, C.byref(self.cfg), C.byref(w.struct), _ptr(self.conv), _ptr(self.h),
               _ptr(x_in), _ptr(residual), self.batch, seqlen, flags, _ptr(ws), ws.numel(), _stream(stream))


class Mamba2Stack:
    """n_layers x [pre-norm RMSNorm (weight 1, reading Q16) -> Mamba-2 mixer -> fp32 residual] on one
    TP rank: chunk-major prefill carrying the caches into CUDA-graph decode (as stack.MixerStack)."""

    def __init__(self, mixer, m2, weights, batch, max_chunk, flags=L.SSM_AR2_INT8, norm_eps=1e-5):
        self.mx, self.m2, self.weights, self.batch, self.flags, self.eps = mixer, m2, weights, batch, flags, norm_eps
        self.layers = [Mamba2Mixer(mixer, m2, batch, max_chunk) for _ in weights]
        ws, wd = self.layers[0].ws, self.layers[0].ws_dec           # one workspace pair for all layers
        for lyr in self.layers[1:]:
            lyr.ws, lyr.ws_dec = ws, wd
        D = m2.d_model
        self.xbuf = torch.empty((batch * max_chunk, D), dtype=torch.bfloat16, device=mixer.device)
        self.xbuf_dec = torch.empty((batch, D), dtype=torch.bfloat16, device=mixer.device)
        self.graph = None
        self.graph_launches = 0
        self._graph_parity = 0

    def reset(self, stream=None):
        for lyr in self.layers:
            lyr.reset()

    def prefill_chunk(self, res, stream=None, h0=None):
        n = res.shape[0]
        x = self.xbuf[:n]
        for w, lyr in zip(self.weights, self.layers):
            self.mx.rmsnorm(res, x, None, self.eps, stream)
            lyr(w, x, res, n // self.batch, self.flags, stream)

    def decode_step(self, res_t, stream=None):
        for w, lyr in zip(self.weights, self.layers):
            self.mx.rmsnorm(res_t, self.xbuf_dec, None, self.eps, stream)
            lyr(w, self.xbuf_dec, res_t, 1, self.flags, stream)

    def capture_decode(self, res_t, probes=(), warmup=True):
        if warmup:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.decode_step(res_t, s)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        before = self.mx.launches()
        self._graph_parity = self.mx.epoch() & 1
        e0 = self.mx.epoch()
        with torch.cuda.graph(g):
            self.decode_step(res_t)
            if (self.mx.epoch() - e0) % 2:
                self.mx.barrier()
        self.graph_launches = self.mx.launches() - before
        self.graph = g
        return g

    def replay(self, graph=None, stream=None):
        if self.mx.tp_size > 1 and (self.mx.epoch() & 1) != self._graph_parity:
            self.mx.barrier(stream)
        (graph or self.graph).replay()


def synthetic_mamba2_layer(m2, layer, seed=5000, device="cuda"):
    """Full Mamba-2 layer weights generated ON the device (the recipe of synth.mamba2_weights) for
    the full-depth bench."""
    import math
    g = torch.Generator(device=device).manual_seed(seed + layer)
    D, E, N, G, K = m2.d_model, m2.d_inner, m2.d_state, m2.n_groups, m2.d_conv
    H = m2.n_heads
    Cd = E + 2 * G * N
    f = dict(device=device, dtype=torch.float32)

    def u(shape, bound):
        return (torch.rand(shape, generator=g, **f) * 2 - 1) * bound
    w = {"w_in": u((2 * E + 2 * G * N + H, D), 1 / math.sqrt(D)), "conv_w": u((Cd, K), 1 / math.sqrt(K)),
         "conv_b": u((Cd,), 1 / math.sqrt(K))}
    lo, hi = math.log(1e-3), math.log(1e-1)
    dt0 = torch.exp(torch.rand((H,), generator=g, **f) * (hi - lo) + lo)
    w["dt_bias"] = dt0 + torch.log(-torch.expm1(-dt0))
    w["a_log"] = torch.log(1.0 + 15.0 * torch.rand((H,), generator=g, **f))
    w["d_skip"] = torch.ones((H,), **f)
    w["norm_w"] = 1.0 + 0.1 * torch.randn((E,), generator=g, **f)
    w["w_out"] = u((D, E), 1 / math.sqrt(E)) / math.sqrt(2.0 * max(m2.n_layers, 1))
    return w
