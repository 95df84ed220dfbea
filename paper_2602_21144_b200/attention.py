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
    def __init__(self, adims, full, tp_size=1, rank=0, device="cuda", shared=None):
        """full: dict of the unsharded block (synth.shared_block_weights layout: norm1, w_q, w_k, w_v,
        w_o, norm2, w_g, w_u, w_d, w_lin).  shared: another SharedBlockWeights whose block tensors
        are reused (Zamba shares one block over its hybrid layers; only w_lin is per layer), in
        which case only full["w_lin"] is read."""
        H, I = adims.n_heads, adims.intermediate
        d = 2 * adims.d_model // H
        hk, ik = H // tp_size, I // tp_size
        rows = slice(rank * hk * d, (rank + 1) * hk * d)
        cols = slice(rank * ik, (rank + 1) * ik)

        def bf(t):
            return t.to(device=device, dtype=torch.bfloat16).contiguous()

        def f32(t):
            return t.to(device=device, dtype=torch.float32).contiguous()

        if shared is not None:
            self.tensors = dict(shared.tensors)
            self.tensors["w_lin"] = bf(full["w_lin"])
            self.struct = L.ssm_attn_weights_t(**{k: v.data_ptr() for k, v in self.tensors.items()})
            return
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

    def __init__(self, mixer, adims, batch, max_seq, max_chunk, stream=None, workspaces=None):
        """workspaces: (prefill, decode) workspaces to share with the other application sites of the
        block (they run one after another), else allocated here."""
        self.mx, self.adims, self.batch = mixer, adims, batch
        self.cfg = L.ssm_attn_config_t(adims.n_heads, adims.intermediate, adims.eps, max_seq)
        nb = C.c_size_t()
        L.call("ssm_kv_bytes", mixer.handle, C.byref(self.cfg), batch, C.byref(nb))
        self.kv_buf = torch.empty(nb.value, dtype=torch.uint8, device=mixer.device)
        self.kv = C.c_void_p()
        L.call("ssm_kv_alloc", mixer.handle, C.byref(self.cfg), batch, _ptr(self.kv_buf), nb.value, _stream(stream),
               C.byref(self.kv))
        self.ws, self.ws_dec = workspaces if workspaces is not None else (self.workspace(max_chunk),
                                                                           self.workspace(1))

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


def synthetic_shared_block(adims, layers, seed=3000, device="cuda"):
    """Full-size shared block generated ON the device (the recipe of synth.shared_block_weights:
    RMSNorm weights 1 + N(0, 0.1), projections U(+-1/sqrt(fan_in)), w_lin / 4), for the bench where
    host generation of ~330M parameters would dominate; returns the block dict (with the first
    layer's w_lin) and {layer: w_lin}."""
    import math
    g = torch.Generator(device=device).manual_seed(seed)
    D, I = adims.d_model, adims.intermediate
    A = 2 * D
    f = dict(device=device, dtype=torch.float32)

    def u(shape, bound, gen=g):
        return (torch.rand(shape, generator=gen, **f) * 2 - 1) * bound

    w = {"norm1": 1.0 + 0.1 * torch.randn((A,), generator=g, **f), "w_q": u((A, A), 1 / math.sqrt(A)),
         "w_k": u((A, A), 1 / math.sqrt(A)), "w_v": u((A, A), 1 / math.sqrt(A)), "w_o": u((D, A), 1 / math.sqrt(A)),
         "norm2": 1.0 + 0.1 * torch.randn((D,), generator=g, **f), "w_g": u((I, D), 1 / math.sqrt(D)),
         "w_u": u((I, D), 1 / math.sqrt(D)), "w_d": u((D, I), 1 / math.sqrt(I))}
    lins = {}
    for li in layers:
        g2 = torch.Generator(device=device).manual_seed(seed + 1 + li)
        lins[li] = u((D, D), 1 / math.sqrt(D), g2) / 4.0
    w["w_lin"] = lins[layers[0]] if layers else u((D, D), 1 / math.sqrt(D)) / 4.0
    return w, lins


def hybrid_config(adims, full, lins, tp_size, rank, max_seq, device="cuda"):
    """MixerStack(hybrid=...) argument: one sharded copy of the shared block, per-layer w_lin."""
    base = None
    weights = {}
    for li, wl in lins.items():
        if base is None:
            base = SharedBlockWeights(adims, dict(full, w_lin=wl), tp_size, rank, device)
            weights[li] = base
        else:
            weights[li] = SharedBlockWeights(adims, {"w_lin": wl}, tp_size, rank, device, shared=base)
    return dict(adims=adims, weights=weights, max_seq=max_seq)
