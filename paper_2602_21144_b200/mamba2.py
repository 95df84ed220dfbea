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
