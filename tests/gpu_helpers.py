"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI and the
oracle on the same seeded inputs, and compare normwise (SURVEY.md §8(c) Q10:
max|gpu - ref| / max|ref| per output tensor)."""
from __future__ import annotations

import numpy as np
import torch

import synth
from paper_2602_21144_b200 import LayerWeights, State, TPMixer, _lib as L

TOL = {"fp32": 1e-5, "bf16": 2e-2}  # north_star tolerances


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def prep_weights(dims, layer, dtype, seed=1000):
    """Full weights (float64 CPU) rounded to the storage precision of the GPU path, so the
    oracle sees exactly the values the kernels see (weight-cast error
    is not counted).  Matrices in the activation dtype, vectors fp32."""
    w = synth.layer_weights(dims, layer, seed)
    mats = ("w_in", "w_x", "w_dt", "w_out")
    out = {}
    for k, v in w.items():
        if k in mats and dtype == "bf16":
            out[k] = synth.bf16_round(v)
        else:
            out[k] = v.to(torch.float32).to(torch.float64)
    return out


def prep_acts(batch, seqlen, dims, dtype, seed=42):
    x, res = synth.activations(batch, seqlen, dims.d_model, seed)
    x = synth.bf16_round(x) if dtype == "bf16" else x.to(torch.float32).to(torch.float64)
    res = res.to(torch.float32).to(torch.float64)
    return x, res


def to_dev(t, dtype):
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    return t.to(dt).cuda().contiguous()


def np64(d):
    return {k: v.numpy() for k, v in d.items()}


def oracle_state_from_gpu_layout(conv, h):
    """GPU conv window [B][K-1][E_k] -> oracle [B][E_k][K-1]."""
    return conv.float().cpu().double().permute(0, 2, 1).numpy(), h.cpu().double().numpy()


from paper_2602_21144_b200.virtual import VirtualGroup  # noqa: E402,F401  (moved into the package)
