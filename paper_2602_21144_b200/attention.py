"""Zamba's shared transformer block on one TP rank: Python
marshalling over ssm_attn_block / ssm_kv_* / ssm_rmsnorm_add (include/ssm_tp.h).  Every step runs
in libssmtp's kernels; PyTorch only allocates the shards, the KV cache and the workspace.

Sharding (reading Z1): rank r owns heads [r H/k, (r+1) H/k) -- rows of W_q, W_k, W_v packed as
q | k | v and the matching columns of W_o -- and MLP columns [r I/k, (r+1) I/k) (rows of W_g, W_u
packed gate | up, columns of W_d); the norms and the hybrid layer's W_lin are replicated."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from .mixer import _ptr, _stream


class SharedBlockWeights:
    def __init__(self, adims, full, tp_size=1, rank=0, device="cuda"):
        """full: dict of the unsharded block (synth.shared_block_weights layout: norm1, w_q, w_k, w_v,
        w_o, norm2, w_g, w_u, w_d, w_lin)."""
        H, I = adims.n_heads, adims.intermediate
        d = 2 * adims.d_model // H
        hk, ik = H // tp_size, I // tp_size
        rows = slice(rank * hk * d, (rank + 1) * hk * d)
        cols = slice(rank * ik, (rank + 1) * ik)

        def bf(t):
            return t.to(device=device, dtype=torch.bfloat16).contiguous()

        def f32(t):
            return t.to(device=device, dtype=torch.float32).contiguous()

        self.tensors = {
            "norm1": f32(full["norm1"]),
            "w_qkv": bf(torch.cat([full["w_q"][rows], full["w_k"][rows], full["w_v"][rows]], 0)),
            "w_o": bf(full["w_o"][:, rows]),
            "norm2": f32(full["norm2"]),
            "w_gu": bf(torch.cat([full["w_g"][cols], full["w_u"][cols]], 0)),
            "w_d": bf(full["w_d"][:, cols]),
            "w_lin": bf(full["w_lin"]),
        }
        self.struct = L.ssm_attn_weights_t(**{k: v.data_ptr() for k, v in self.tensors.items()})


class SharedBlock:
    """One application site of the shared block (its KV cache) on this rank of `mixer`."""

    def __init__(self, mixer, adims, batch, max_seq, max_chunk, stream=None):
        self.mx, self.adims, self.batch = mixer, adims, batch
        self.cfg = L.ssm_attn_config_t(adims.n_heads, adims.intermediate, adims.eps, max_seq)
        nb = C.c_size_t()
        L.call("ssm_kv_bytes", mixer.handle, C.byref(self.cfg), batch, C.byref(nb))
        self.kv_buf = torch.empty(nb.value, dtype=torch.uint8, device=mixer.device)
        self.kv = C.c_void_p()
        L.call("ssm_kv_alloc", mixer.handle, C.byref(self.cfg), batch, _ptr(self.kv_buf), nb.value, _stream(stream),
               C.byref(self.kv))
        self.ws = self.workspace(max_chunk)
        self.ws_dec = self.workspace(1)

    def workspace(self, seqlen):
        nb = C.c_size_t()
        L.call("ssm_attn_workspace_bytes", self.mx.handle, C.byref(self.cfg), self.batch, seqlen, C.byref(nb))
        return torch.empty(max(nb.value, 256), dtype=torch.uint8, device=self.mx.device)

    def reset(self, stream=None):
        L.call("ssm_kv_reset", self.kv, _stream(stream))

    def __call__(self, w, h, h0, t_out, seqlen, flags=0, stream=None):
        """t_out [batch*seqlen, D] fp32 := block(h, h0); this call's K, V appended to the cache."""
        ws = self.ws_dec if seqlen == 1 else self.ws
        L.call("ssm_attn_block", self.mx.handle, C.byref(self.cfg), C.byref(w.struct), self.kv, _ptr(h), _ptr(h0),
               _ptr(t_out), self.batch, seqlen, flags, _ptr(ws), ws.numel(), _stream(stream))

    def __del__(self):
        try:
            if self.kv:
                L.LIB.ssm_kv_free(self.kv)
        except Exception:
            pass
