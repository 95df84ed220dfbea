"""ctypes binding of libssmtp.so (include/ssm_tp.h).  Argument marshalling only:
every step of the mixer runs in the library's CUDA kernels.  There is no CPU or
alternative-backend path: if the shared library is missing, importing the binding
raises."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libssmtp.so")

SSM_BF16, SSM_FP32 = 0, 1
SSM_AR2_INT8, SSM_AR2_FP32, SSM_AR2_EXTERNAL, SSM_AR2_FP16 = 0x1, 0x2, 0x4, 0x8
SSM_QAR_ACCUMULATE, SSM_QAR_FP16, SSM_QAR_TWOSHOT, SSM_QAR_ONESHOT = 0x10, 0x20, 0x40, 0x80
SSM_DECODE_UNFUSED, SSM_AR2_BF16, SSM_QAR_BF16, SSM_TP_NAIVE, SSM_QAR_REQUANT = 0x100, 0x200, 0x400, 0x1000, 0x2000
SSM_QAR_FP32 = 0x4000
SSM_COMM_VIRTUAL = 0x1

STATUS = {0: "SSM_OK", 1: "SSM_ERR_ARG", 2: "SSM_ERR_DIM", 3: "SSM_ERR_SHARD", 4: "SSM_ERR_RANK",
          5: "SSM_ERR_CACHE", 6: "SSM_ERR_PROTOCOL", 7: "SSM_ERR_CUDA", 8: "SSM_ERR_UNSUPPORTED"}


class SSMError(RuntimeError):
    def __init__(self, code, func, msg):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"{func}: {self.name}: {msg}")


class ssm_config_t(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("d_inner", C.c_int32), ("d_state", C.c_int32), ("d_conv", C.c_int32),
                ("dt_rank", C.c_int32), ("n_heads", C.c_int32), ("dtype", C.c_int32), ("bcdt_rmsnorm", C.c_int32),
                ("rms_eps", C.c_float), ("qar_block", C.c_int32)]


class ssm_comm_t(C.Structure):
    _fields_ = [("rank", C.c_int32), ("tp_size", C.c_int32), ("peer_bufs", C.POINTER(C.c_void_p)),
                ("buf_bytes", C.c_size_t), ("flags", C.c_int32)]


class ssm_layer_weights_t(C.Structure):
    _fields_ = [("w_in", C.c_void_p), ("conv_w", C.c_void_p), ("conv_b", C.c_void_p), ("w_x", C.c_void_p),
                ("w_dt", C.c_void_p), ("b_dt", C.c_void_p), ("a_log", C.c_void_p), ("d_skip", C.c_void_p),
                ("w_out", C.c_void_p), ("w_in_pk", C.c_void_p), ("w_x_pk", C.c_void_p), ("w_out_pk", C.c_void_p),
                ("w_in_naive", C.c_void_p)]


class ssm_attn_config_t(C.Structure):
    _fields_ = [("n_heads", C.c_int32), ("intermediate", C.c_int32), ("eps", C.c_float), ("max_seq", C.c_int32)]


class ssm_attn_weights_t(C.Structure):
    _fields_ = [("norm1", C.c_void_p), ("w_qkv", C.c_void_p), ("w_o", C.c_void_p), ("norm2", C.c_void_p),
                ("w_gu", C.c_void_p), ("w_d", C.c_void_p), ("w_lin", C.c_void_p)]


class ssm_m2_config_t(C.Structure):
    _fields_ = [("d_inner", C.c_int32), ("d_state", C.c_int32), ("headdim", C.c_int32), ("n_groups", C.c_int32),
                ("d_conv", C.c_int32), ("eps", C.c_float)]


class ssm_m2_weights_t(C.Structure):
    _fields_ = [("w_in", C.c_void_p), ("conv_w", C.c_void_p), ("conv_b", C.c_void_p), ("dt_bias", C.c_void_p),
                ("a_log", C.c_void_p), ("d_skip", C.c_void_p), ("norm_w", C.c_void_p), ("w_out", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libssmtp.so not built ({LIB_PATH}); run `python -m paper_2602_21144_b200.build`")
    lib = C.CDLL(LIB_PATH)
    st = C.c_int
    vp, sz, i32, i64 = C.c_void_p, C.c_size_t, C.c_int32, C.c_int64
    P = C.POINTER
    sig = {
        "ssm_last_error": (C.c_char_p, []),
        "ssm_version": (C.c_char_p, []),
        "ssm_tp_init": (st, [P(ssm_config_t), P(ssm_comm_t), P(vp)]),
        "ssm_tp_destroy": (st, [vp]),
        "ssm_comm_bytes": (st, [P(ssm_config_t), i32, i64, P(sz)]),
        "ssm_workspace_bytes": (st, [vp, i32, i32, P(sz)]),
        "ssm_workspace_bytes_flags": (st, [vp, i32, i32, C.c_uint32, P(sz)]),
        "ssm_state_bytes": (st, [vp, i32, P(sz), P(sz)]),
        "ssm_state_alloc": (st, [vp, i32, vp, sz, vp, sz, vp, P(vp)]),
        "ssm_state_reset": (st, [vp, vp]),
        "ssm_state_free": (st, [vp]),
        "ssm_mixer_prefill": (st, [vp, P(ssm_layer_weights_t), vp, vp, vp, i32, i32, C.c_uint32, vp, sz, vp]),
        "ssm_mixer_prefill_normed": (st, [vp, P(ssm_layer_weights_t), vp, vp, vp, C.c_float, vp, vp, vp, i32, i32,
                                          C.c_uint32, vp, sz, vp]),
        "ssm_rowstats": (st, [vp, vp, vp, vp, i64, vp]),
        "ssm_mixer_decode": (st, [vp, P(ssm_layer_weights_t), vp, vp, vp, i32, C.c_uint32, vp, sz, vp]),
        "ssm_mixer_decode_block": (st, [vp, P(ssm_layer_weights_t), vp, vp, i32, C.c_float, C.c_uint32, vp, sz, vp]),
        "ssm_qallreduce": (st, [vp, vp, vp, sz, C.c_uint32, vp]),
        "ssm_rmsnorm": (st, [vp, vp, vp, C.c_float, vp, i64, vp]),
        "ssm_tp_check": (st, [vp, vp]),
        "ssm_rmsnorm_add": (st, [vp, vp, vp, vp, C.c_float, vp, i64, vp]),
        "ssm_m2_state_bytes": (st, [vp, P(ssm_m2_config_t), i32, P(sz), P(sz)]),
        "ssm_m2_workspace_bytes": (st, [vp, P(ssm_m2_config_t), i32, i32, P(sz)]),
        "ssm_m2_mixer": (st, [vp, P(ssm_m2_config_t), P(ssm_m2_weights_t), vp, vp, vp, vp, i32, i32, C.c_uint32, vp,
                              sz, vp]),
        "ssm_kv_bytes": (st, [vp, P(ssm_attn_config_t), i32, P(sz)]),
        "ssm_kv_alloc": (st, [vp, P(ssm_attn_config_t), i32, vp, sz, vp, P(vp)]),
        "ssm_kv_reset": (st, [vp, vp]),
        "ssm_kv_free": (st, [vp]),
        "ssm_attn_workspace_bytes": (st, [vp, P(ssm_attn_config_t), i32, i32, P(sz)]),
        "ssm_attn_block": (st, [vp, P(ssm_attn_config_t), P(ssm_attn_weights_t), vp, vp, vp, vp, i32, i32, C.c_uint32,
                                vp, sz, vp]),
        "ssm_tp_stats": (st, [vp, P(i64), P(i64)]),
        "ssm_tp_launch_count": (st, [vp, P(i64)]),
        "ssm_tp_epoch": (st, [vp, P(C.c_uint32)]),
        "ssm_tp_barrier": (st, [vp, vp]),
        "ssm_tp_fused_calls": (st, [vp, P(i64)]),
        "ssm_tp_probe": (st, [vp, i32, i32]),
        "ssm_tp_probe_read": (st, [vp, i32, P(C.c_float), i32, P(i32)]),
        "ssm_dbg_gemm": (st, [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp]),
        "ssm_dbg_set_gemm_pair": (st, [i32]),
        "ssm_packed_weight_bytes": (st, [i32, i32, P(sz)]),
        "ssm_pack_weight": (st, [vp, vp, i32, i32, vp, sz, vp]),
        "ssm_dbg_gemm_packed": (st, [vp, vp, vp, vp, vp, i32, i32, i32, i32, vp]),
        "ssm_dbg_gemm_ld": (st, [vp, vp, i64, vp, i64, vp, i32, i32, i32, i32, i32, vp]),
        "ssm_dbg_scan": (st, [vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, i32, i32, vp]),
        "ssm_dstack_bytes": (st, [vp, i32, i32, i32, P(sz)]),
        "ssm_dstack_create": (st, [vp, i32, P(ssm_layer_weights_t), P(vp), i32, C.c_float, i32, vp, sz, vp, P(vp)]),
        "ssm_dstack_decode": (st, [vp, vp, vp]),
        "ssm_dstack_destroy": (st, [vp]),
        "ssm_dbg_dstack_trace": (st, [vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = _load()
EXPORTED = ["ssm_last_error", "ssm_version", "ssm_tp_init", "ssm_tp_destroy", "ssm_comm_bytes", "ssm_workspace_bytes",
            "ssm_workspace_bytes_flags",
            "ssm_state_bytes", "ssm_state_alloc", "ssm_state_reset", "ssm_state_free", "ssm_mixer_prefill",
            "ssm_mixer_prefill_normed", "ssm_rowstats",
            "ssm_mixer_decode", "ssm_mixer_decode_block", "ssm_qallreduce", "ssm_rmsnorm", "ssm_tp_check", "ssm_tp_stats", "ssm_tp_epoch",
            "ssm_tp_barrier", "ssm_tp_launch_count", "ssm_tp_fused_calls", "ssm_tp_probe", "ssm_tp_probe_read",
            "ssm_packed_weight_bytes", "ssm_pack_weight", "ssm_dbg_gemm", "ssm_dbg_set_gemm_pair", "ssm_dbg_gemm_packed", "ssm_dbg_gemm_ld",
            "ssm_dbg_scan", "ssm_rmsnorm_add", "ssm_kv_bytes", "ssm_kv_alloc", "ssm_kv_reset", "ssm_kv_free",
            "ssm_attn_workspace_bytes", "ssm_attn_block", "ssm_m2_state_bytes", "ssm_m2_workspace_bytes",
            "ssm_m2_mixer", "ssm_dstack_bytes", "ssm_dstack_create", "ssm_dstack_decode", "ssm_dstack_destroy",
            "ssm_dbg_dstack_trace"]
PROBE = {"in_proj": 1, "conv": 2, "x_proj": 3, "dt_proj": 4, "scan": 5, "out_proj": 6, "ar2": 7, "decode_step": 8,
         "in_proj_decode": 9}


def check(rc, func):
    if rc != 0:
        raise SSMError(rc, func, LIB.ssm_last_error().decode())


def call(name, *args):
    check(getattr(LIB, name)(*args), name)


def make_config(dims, dtype="bf16", qar_block=128):
    """dims: any object with d_model, d_inner, d_state, d_conv, dt_rank, n_heads, bcdt_rmsnorm, rms_eps."""
    c = ssm_config_t()
    c.d_model, c.d_inner, c.d_state = dims.d_model, dims.d_inner, dims.d_state
    c.d_conv, c.dt_rank, c.n_heads = dims.d_conv, dims.dt_rank, getattr(dims, "n_heads", 1)
    c.dtype = SSM_BF16 if dtype == "bf16" else SSM_FP32
    c.bcdt_rmsnorm = int(bool(getattr(dims, "bcdt_rmsnorm", False)))
    c.rms_eps = float(getattr(dims, "rms_eps", 1e-6))
    c.qar_block = min(qar_block, dims.d_model)
    return c


def comm_bytes(cfg, tp_size, max_tokens):
    out = C.c_size_t()
    call("ssm_comm_bytes", C.byref(cfg), tp_size, max_tokens, C.byref(out))
    return out.value
