"""Python API over the C ABI: one rank's TP mixer handle, weight shards, SSM cache.

PyTorch is used only for device memory and streams; every step of the mixer runs
in libssmtp's CUDA kernels (include/ssm_tp.h).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from ._lib import SSMError  # noqa: F401  (re-export)


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def channel_range(d_inner, tp_size, rank):
    """[lo, hi) of d_inner owned by `rank` (each GPU owns a disjoint
    contiguous channel slice).  Raises SSMError(SSM_ERR_SHARD / SSM_ERR_RANK)."""
    if tp_size < 1 or d_inner % tp_size:
        raise SSMError(3, "channel_range", f"d_inner={d_inner} not divisible by tp={tp_size}")
    if not 0 <= rank < tp_size:
        raise SSMError(4, "channel_range", f"rank {rank} not in [0,{tp_size})")
    ek = d_inner // tp_size
    return rank * ek, (rank + 1) * ek


class LayerWeights:
    """Rank-local shard of one mixer layer, resident on the device.

    The channel splitter (§4.2) and packed-parameter placement
    (§4.3): the packed in_proj is sliced per logical field
    (the rank's x rows and its z rows, never across the packed boundary); conv,
    dt_proj, b_dt, A_log and D rows follow the channels; x_proj and out_proj are
    sliced by input columns (row-parallel partials).  Zamba heads: the rank's
    x_proj is block-diagonal over the heads it touches.
    """

    def __init__(self, dims, full, tp_size=1, rank=0, dtype="bf16", device="cuda", naive=False):
        lo, hi = channel_range(dims.d_inner, tp_size, rank)
        E, H = dims.d_inner, dims.n_heads
        Eh = E // H
        mat = torch.bfloat16 if dtype == "bf16" else torch.float32
        f32 = torch.float32

        def dev(t, dt):
            return t.to(device=device, dtype=dt).contiguous()

        w_in = torch.cat([full["w_in"][lo:hi], full["w_in"][E + lo:E + hi]], 0)
        heads = [h for h in range(H) if max(lo, h * Eh) < min(hi, (h + 1) * Eh)]
        P = dims.dt_rank + 2 * dims.d_state
        w_x = torch.zeros((len(heads) * P, hi - lo), dtype=full["w_x"].dtype)
        for j, h in enumerate(heads):
            a, b = max(lo, h * Eh), min(hi, (h + 1) * Eh)
            w_x[j * P:(j + 1) * P, a - lo:b - lo] = full["w_x"][h][:, a - h * Eh:b - h * Eh]
        self.tensors = {
            "w_in": dev(w_in, mat),
            "conv_w": dev(full["conv_w"][lo:hi], f32),
            "conv_b": dev(full["conv_b"][lo:hi], f32),
            "w_x": dev(w_x, mat),
            "w_dt": dev(full["w_dt"][lo:hi], mat),
            "b_dt": dev(full["b_dt"][lo:hi], f32),
            "a_log": dev(full["a_log"][lo:hi], f32),
            "d_skip": dev(full["d_skip"][lo:hi], f32),
            "w_out": dev(full["w_out"][:, lo:hi], mat),
        }
        if naive:  # the naive baseline's uniform split of the PACKED in_proj (SSM_TP_NAIVE)
            wn = 2 * E // tp_size
            self.tensors["w_in_naive"] = dev(full["w_in"][rank * wn:(rank + 1) * wn], mat)
        self.struct = L.ssm_layer_weights_t(**{k: v.data_ptr() for k, v in self.tensors.items()})

    def pack(self, mixer, stream=None):
        """Pre-tile w_in, w_x, w_out (ssm_pack_weight) so decode streams contiguous 16 KB tiles."""
        for name in ("w_in", "w_x", "w_out"):
            t = self.tensors[name]
            rows, cols = t.shape
            nb = C.c_size_t()
            L.call("ssm_packed_weight_bytes", rows, cols, C.byref(nb))
            pk = torch.empty(nb.value // 2, dtype=torch.bfloat16, device=t.device)
            L.call("ssm_pack_weight", mixer.handle, _ptr(t), rows, cols, _ptr(pk), nb.value, _stream(stream))
            self.tensors[name + "_pk"] = pk
            setattr(self.struct, name + "_pk", pk.data_ptr())
        return self


class State:
    """SSM cache of one layer on this rank: conv window + fp32 h."""

    def __init__(self, mixer, batch, stream=None):
        cb, hb = C.c_size_t(), C.c_size_t()
        L.call("ssm_state_bytes", mixer.handle, batch, C.byref(cb), C.byref(hb))
        dt = torch.bfloat16 if mixer.dtype == "bf16" else torch.float32
        ek, K, N = mixer.ek, mixer.dims.d_conv, mixer.dims.d_state
        self.conv = torch.empty((batch, K - 1, ek), dtype=dt, device=mixer.device)
        # h [batch][E_k][N] fp32 followed by the library's decode accumulator (same buffer)
        self._hbuf = torch.empty(hb.value // 4, dtype=torch.float32, device=mixer.device)
        self.h = self._hbuf[:batch * ek * N].view(batch, ek, N)
        self.handle = C.c_void_p()
        L.call("ssm_state_alloc", mixer.handle, batch, _ptr(self.conv), cb.value, _ptr(self._hbuf), hb.value,
               _stream(stream), C.byref(self.handle))
        self.batch = batch

    def reset(self, stream=None):
        L.call("ssm_state_reset", self.handle, _stream(stream))

    def __del__(self):
        try:
            if self.handle:
                L.LIB.ssm_state_free(self.handle)
        except Exception:
            pass


class TPMixer:
    """Handle of one rank (ssm_tp_t).  peer_bufs: list of device pointers (ints) of the
    symmetric buffers of all ranks (None for tp_size == 1)."""

    def __init__(self, dims, dtype="bf16", rank=0, tp_size=1, peer_bufs=None, buf_bytes=0, virtual=False,
                 qar_block=128, device="cuda"):
        self.dims, self.dtype, self.rank, self.tp_size = dims, dtype, rank, tp_size
        self.device = torch.device(device)
        self.cfg = L.make_config(dims, dtype, qar_block)
        self.ek = dims.d_inner // tp_size if tp_size > 0 and dims.d_inner % tp_size == 0 else 0
        comm = L.ssm_comm_t()
        comm.rank, comm.tp_size = rank, tp_size
        self._peer_arr = None
        if peer_bufs is not None:
            self._peer_arr = (C.c_void_p * len(peer_bufs))(*peer_bufs)
            comm.peer_bufs = C.cast(self._peer_arr, C.POINTER(C.c_void_p))
        comm.buf_bytes = buf_bytes
        comm.flags = L.SSM_COMM_VIRTUAL if virtual else 0
        self.handle = C.c_void_p()
        L.call("ssm_tp_init", C.byref(self.cfg), C.byref(comm), C.byref(self.handle))

    def __del__(self):
        try:
            if self.handle:
                L.LIB.ssm_tp_destroy(self.handle)
        except Exception:
            pass

    # ---- sizes
    def workspace_bytes(self, batch, seqlen, flags=0):
        out = C.c_size_t()
        L.call("ssm_workspace_bytes_flags", self.handle, batch, seqlen, flags, C.byref(out))
        return out.value

    def workspace(self, batch, seqlen, flags=0):
        n = self.workspace_bytes(batch, seqlen, flags)
        return torch.empty(max(n, 256), dtype=torch.uint8, device=self.device)

    # ---- compute
    def prefill(self, w, state, x_in, residual, flags=L.SSM_AR2_INT8, workspace=None, stream=None):
        B, Lq = state.batch, x_in.numel() // (state.batch * self.dims.d_model)
        ws = workspace if workspace is not None else self.workspace(B, Lq)
        L.call("ssm_mixer_prefill", self.handle, C.byref(w.struct), state.handle, _ptr(x_in), _ptr(residual), B, Lq,
               flags, _ptr(ws), ws.numel(), _stream(stream))

    def prefill_normed(self, w, state, x_in, ss_in, residual, x_next=None, ss_next=None, norm_eps=1e-5,
                       flags=L.SSM_AR2_INT8, workspace=None, stream=None):
        """One pre-norm prefill block with the norm folded around the projections
        (ssm_mixer_prefill_normed): x_in = bf16(residual), ss_in its row sums of squares; the out_proj
        epilogue writes x_next / ss_next for the next layer."""
        B, Lq = state.batch, x_in.numel() // (state.batch * self.dims.d_model)
        ws = workspace if workspace is not None else self.workspace(B, Lq)
        L.call("ssm_mixer_prefill_normed", self.handle, C.byref(w.struct), state.handle, _ptr(x_in), _ptr(ss_in),
               C.c_float(norm_eps), _ptr(residual), _ptr(x_next), _ptr(ss_next), B, Lq, flags, _ptr(ws), ws.numel(),
               _stream(stream))

    def rowstats(self, residual, x_out, ss_out, stream=None):
        """x_out = bf16(residual), ss_out = row sums of squares (ssm_rowstats)."""
        L.call("ssm_rowstats", self.handle, _ptr(residual), _ptr(x_out), _ptr(ss_out),
               residual.numel() // self.dims.d_model, _stream(stream))

    def decode(self, w, state, x_in, residual, flags=L.SSM_AR2_INT8, workspace=None, stream=None):
        B = state.batch
        ws = workspace if workspace is not None else self.workspace(B, 1)
        L.call("ssm_mixer_decode", self.handle, C.byref(w.struct), state.handle, _ptr(x_in), _ptr(residual), B, flags,
               _ptr(ws), ws.numel(), _stream(stream))

    def decode_block(self, w, state, residual, norm_eps=1e-5, flags=L.SSM_AR2_INT8, workspace=None, stream=None):
        """One pre-norm decode block: residual += mixer(RMSNorm(residual)) (ssm_mixer_decode_block)."""
        B = state.batch
        ws = workspace if workspace is not None else self.workspace(B, 1)
        L.call("ssm_mixer_decode_block", self.handle, C.byref(w.struct), state.handle, _ptr(residual), B,
               C.c_float(norm_eps), flags, _ptr(ws), ws.numel(), _stream(stream))

    def qallreduce(self, partial, out, accumulate=False, stream=None, fp16=False, twoshot=False, bf16=False,
                   requant=False):
        """fp16=True: the paper's FP32 -> FP16 wire instead of int8 blocks;
        bf16=True: the custom bf16 wire; twoshot / requant: the int8 two-shot schedules."""
        L.call("ssm_qallreduce", self.handle, _ptr(partial), _ptr(out), partial.numel(),
               (L.SSM_QAR_ACCUMULATE if accumulate else 0) | (L.SSM_QAR_FP16 if fp16 else 0) |
               (L.SSM_QAR_BF16 if bf16 else 0) | (L.SSM_QAR_TWOSHOT if twoshot else 0) |
               (L.SSM_QAR_REQUANT if requant else 0), _stream(stream))

    def rmsnorm(self, residual, out, weight=None, eps=1e-5, stream=None):
        L.call("ssm_rmsnorm", self.handle, _ptr(residual), _ptr(weight), C.c_float(eps), _ptr(out),
               residual.numel() // self.dims.d_model, _stream(stream))

    def rmsnorm_add(self, a, b, out, weight=None, eps=1e-5, stream=None):
        """out = RMSNorm(a + b) * weight (b may be None): the hybrid layer's Mamba pre-norm."""
        L.call("ssm_rmsnorm_add", self.handle, _ptr(a), _ptr(b), _ptr(weight), C.c_float(eps), _ptr(out),
               a.numel() // self.dims.d_model, _stream(stream))

    def check(self, stream=None):
        L.call("ssm_tp_check", self.handle, _stream(stream))

    def stats(self):
        a, b = C.c_int64(), C.c_int64()
        L.call("ssm_tp_stats", self.handle, C.byref(a), C.byref(b))
        return {"allreduce": a.value, "bytes_sent": b.value}

    def epoch(self):
        """Collectives enqueued so far (ssm_tp_epoch); collective e uses symmetric half e & 1."""
        e = C.c_uint32()
        L.call("ssm_tp_epoch", self.handle, C.byref(e))
        return e.value

    def barrier(self, stream=None):
        """Payload-free cross-rank barrier (a collective); advances the epoch by one at TP > 1."""
        L.call("ssm_tp_barrier", self.handle, _stream(stream))

    def fused_calls(self):
        """Decode calls that ran the fused in_proj (+conv +x_proj) kernel."""
        n = C.c_int64()
        L.call("ssm_tp_fused_calls", self.handle, C.byref(n))
        return n.value

    def launches(self):
        n = C.c_int64()
        L.call("ssm_tp_launch_count", self.handle, C.byref(n))
        return n.value

    def probe(self, kernel, capacity):
        """Record per-launch CUDA events around `kernel` ('in_proj', 'scan', 'in_proj_decode', ...);
        capacity 0 disables that kind."""
        L.call("ssm_tp_probe", self.handle, L.PROBE[kernel], capacity)

    def probe_read(self, kernel, capacity=100000):
        buf = (C.c_float * capacity)()
        n = C.c_int32()
        L.call("ssm_tp_probe_read", self.handle, L.PROBE[kernel], buf, capacity, C.byref(n))
        return list(buf[:n.value])

    # ---- test-only
    def dbg_gemm(self, A, B, C_out, swap_ab=False, ksplit=1, stream=None):
        M, K = A.shape
        N = B.shape[0]
        L.call("ssm_dbg_gemm", self.handle, _ptr(A), _ptr(B), _ptr(C_out), M, N, K, int(swap_ab), ksplit,
               _stream(stream))

    def dbg_gemm_packed(self, X, W, Wpk, C_out, ksplit=1, stream=None):
        M, K = X.shape
        N = W.shape[0]
        L.call("ssm_dbg_gemm_packed", self.handle, _ptr(X), _ptr(W), _ptr(Wpk), _ptr(C_out), M, N, K, ksplit,
               _stream(stream))

    def pack_weight(self, W, stream=None):
        rows, cols = W.shape
        nb = C.c_size_t()
        L.call("ssm_packed_weight_bytes", rows, cols, C.byref(nb))
        pk = torch.empty(nb.value // 2, dtype=torch.bfloat16, device=W.device)
        L.call("ssm_pack_weight", self.handle, _ptr(W), rows, cols, _ptr(pk), nb.value, _stream(stream))
        return pk

    def dbg_gemm_ld(self, A, B, C_out, M, N, K, swap_ab=False, ksplit=1, stream=None):
        """A [M, K] with row stride A.stride(0), B [N, K] with row stride B.stride(0)."""
        L.call("ssm_dbg_gemm_ld", self.handle, _ptr(A), A.stride(0), _ptr(B), B.stride(0), _ptr(C_out), M, N, K,
               int(swap_ab), ksplit, _stream(stream))

    def dbg_scan(self, u, delta, z, ldz, BC, a_log, d_skip, h, g, batch, seqlen, stream=None):
        L.call("ssm_dbg_scan", self.handle, _ptr(u), _ptr(delta), _ptr(z), ldz, _ptr(BC), _ptr(a_log), _ptr(d_skip),
               _ptr(h), _ptr(g), batch, seqlen, _stream(stream))
