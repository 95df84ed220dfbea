"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no projection, conv, scan,
gate or quantisation).  It only draws seeded random weights and activations
with the value ranges of the Mamba initialisation (SURVEY.md §8(d) "Synthetic
inputs"), and names the model dimensions of the configs in BASELINE.json.
Dimensions not stated by the paper come from the public HF configs
(SURVEY.md §8 config table, C12): expand 2 -> E = 2D, d_conv 4,
dt_rank = ceil(D/16), d_state 16.

Everything is generated with a CPU ``torch.Generator`` so the stream is the
same on every machine; callers move tensors to the device themselves.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict

import torch


@dataclass(frozen=True)
class MixerDims:
    d_model: int
    d_inner: int
    d_state: int = 16
    d_conv: int = 4
    dt_rank: int = 0
    n_heads: int = 1          # x_proj groups: 1 (Mamba, Falcon) or 2 (Zamba)
    bcdt_rmsnorm: bool = False  # Falcon-Mamba weightless RMSNorm on dt/B/C
    rms_eps: float = 1e-6
    n_layers: int = 1

    @property
    def P(self) -> int:
        """Packed x_proj width per head: R + 2N."""
        return self.dt_rank + 2 * self.d_state

    def asdict(self):
        return asdict(self)


def _dims(d_model, n_layers, **kw):
    return MixerDims(d_model=d_model, d_inner=2 * d_model,
                     dt_rank=kw.pop("dt_rank", math.ceil(d_model / 16)),
                     n_layers=n_layers, **kw)


# BASELINE.json configs[0..4]; SURVEY.md §8 config table.
CONFIGS = {
    # cfg1: tiny single layer (SPEC.md:457 dt_rank=4)
    "tiny": MixerDims(d_model=64, d_inner=128, d_state=16, d_conv=4, dt_rank=4, n_layers=1),
    # cfg2/cfg5: Mamba-2.8B
    "mamba2.8b": _dims(2560, 64),
    # cfg3: Falcon-Mamba-7B (dt/B/C RMSNorm on for "Falcon-shaped" runs)
    "falcon7b": _dims(4096, 64, bcdt_rmsnorm=True),
    # cfg4: Zamba-7B Mamba layers (2 mixer heads, dt_rank 232)
    "zamba7b": _dims(3712, 76, dt_rank=232, n_heads=2),
}

# Workloads (batch, prompt, decode) per BASELINE.json configs.
WORKLOADS = {
    "tiny": dict(batch=2, prompt=64, decode=16),
    "mamba2.8b": dict(batch=16, prompt=2048, decode=256),
    "falcon7b": dict(batch=32, prompt=8192, decode=512),
    "zamba7b": dict(batch=16, prompt=4096, decode=512),
    "mamba2.8b-long": dict(batch=8, prompt=65536, decode=256),
}


def _u(g, shape, bound):
    return (torch.rand(shape, generator=g, dtype=torch.float64) * 2.0 - 1.0) * bound


def layer_weights(dims: MixerDims, layer: int = 0, seed: int = 1000) -> dict:
    """Full (unsharded) weights of one mixer layer, float64 CPU tensors.

    Layouts (nn.Linear [out, in]):
      w_in   [2E, D]      rows [0,E) = x path, [E,2E) = z (gate) path
      conv_w [E, K]       tap K-1 multiplies the current token
      conv_b [E]
      w_x    [H, P, E/H]  per head; rows [0,R)=dt, [R,R+N)=B, [R+N,R+2N)=C
      w_dt   [E, R]       channel d uses its head's dt slice
      b_dt   [E]
      a_log  [E, N]       A = -exp(a_log)
      d_skip [E]
      w_out  [D, E]
    """
    g = torch.Generator().manual_seed(seed + layer)
    D, E, N, K, R, H = dims.d_model, dims.d_inner, dims.d_state, dims.d_conv, dims.dt_rank, dims.n_heads
    Eh = E // H
    w = {}
    w["w_in"] = _u(g, (2 * E, D), 1.0 / math.sqrt(D))
    w["conv_w"] = _u(g, (E, K), 1.0 / math.sqrt(K))
    w["conv_b"] = _u(g, (E,), 1.0 / math.sqrt(K))
    w["w_x"] = _u(g, (H, R + 2 * N, Eh), 1.0 / math.sqrt(Eh))
    w["w_dt"] = _u(g, (E, R), 1.0 / math.sqrt(R))
    # Mamba dt init: dt0 ~ logU[1e-3, 1e-1]; bias = inverse-softplus(dt0)
    lo, hi = math.log(1e-3), math.log(1e-1)
    dt0 = torch.exp(torch.rand((E,), generator=g, dtype=torch.float64) * (hi - lo) + lo)
    w["b_dt"] = dt0 + torch.log(-torch.expm1(-dt0))
    # S4D-real A = -(n+1), jittered so no structured-A shortcut applies
    n = torch.arange(1, N + 1, dtype=torch.float64)
    w["a_log"] = torch.log(n)[None, :].expand(E, N) + 0.05 * torch.randn((E, N), generator=g, dtype=torch.float64)
    w["d_skip"] = torch.ones((E,), dtype=torch.float64)
    w["w_out"] = _u(g, (D, E), 1.0 / math.sqrt(E)) / math.sqrt(2.0 * max(dims.n_layers, 1))
    return w


def activations(batch: int, seqlen: int, d_model: int, seed: int = 42):
    """(x_in, residual): normalised-scale inputs ~N(0,1), float64 CPU."""
    g = torch.Generator().manual_seed(seed)
    x = torch.randn((batch, seqlen, d_model), generator=g, dtype=torch.float64)
    res = torch.randn((batch, seqlen, d_model), generator=g, dtype=torch.float64)
    return x, res


def partials(k: int, n: int, seed: int = 7, scale: float = 1.0):
    """k rank-partials of length n for all-reduce tests (float32-representable)."""
    g = torch.Generator().manual_seed(seed)
    return (torch.randn((k, n), generator=g, dtype=torch.float64) * scale).to(torch.float32)


def bf16_round(t: torch.Tensor) -> torch.Tensor:
    """Round to bf16 and back to float64 (input preparation for bf16-mode parity)."""
    return t.to(torch.bfloat16).to(torch.float64)


# ---------------------------------------------------------------------------------------------
# Zamba's shared transformer block: dimensions and seeded weights.
@dataclass(frozen=True)
class AttnDims:
    d_model: int            # D; the block's input is concat(h, h0): 2 D
    n_heads: int            # H; head_dim = 2 D / H
    intermediate: int       # MLP width I
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return 2 * self.d_model // self.n_heads


# Zamba-7B (HF ZambaConfig defaults): hidden 3712, attention hidden 7424, 16 heads of 464, MLP 14848,
# GELU, hybrid (shared-attention) layers at these indices of the 76
ZAMBA7B_ATTN = AttnDims(d_model=3712, n_heads=16, intermediate=14848)
ZAMBA7B_HYBRID_LAYERS = (2, 7, 13, 19, 25, 31, 37, 43, 49, 55, 61, 67, 73)


def shared_block_weights(adims: AttnDims, seed: int = 3000, layer: int = 0) -> dict:
    """Weights of the shared block (float64 CPU; nn.Linear [out, in]) plus one hybrid layer's
    linear (seed + layer): RMSNorm weights 1 + N(0, 0.1) (so a dropped weight shows), the
    projections U(+-1/sqrt(fan_in)), w_lin scaled by 1/4 (the block's output is added to the
    Mamba layer's input)."""
    g = torch.Generator().manual_seed(seed)
    D, H, I = adims.d_model, adims.n_heads, adims.intermediate
    A = 2 * D
    w = {"norm1": 1.0 + 0.1 * torch.randn((A,), generator=g, dtype=torch.float64),
         "w_q": _u(g, (A, A), 1.0 / math.sqrt(A)), "w_k": _u(g, (A, A), 1.0 / math.sqrt(A)),
         "w_v": _u(g, (A, A), 1.0 / math.sqrt(A)), "w_o": _u(g, (D, A), 1.0 / math.sqrt(A)),
         "norm2": 1.0 + 0.1 * torch.randn((D,), generator=g, dtype=torch.float64),
         "w_g": _u(g, (I, D), 1.0 / math.sqrt(D)), "w_u": _u(g, (I, D), 1.0 / math.sqrt(D)),
         "w_d": _u(g, (D, I), 1.0 / math.sqrt(I))}
    g2 = torch.Generator().manual_seed(seed + 1 + layer)
    w["w_lin"] = _u(g2, (D, D), 1.0 / math.sqrt(D)) / 4.0
    return w


# ---------------------------------------------------------------------------------------------
# Mamba-2 (SSD) mixer: dimensions and seeded weights.
@dataclass(frozen=True)
class Mamba2Dims:
    d_model: int
    d_inner: int
    d_state: int = 128
    headdim: int = 64
    n_groups: int = 1
    d_conv: int = 4
    eps: float = 1e-5
    n_layers: int = 1

    @property
    def n_heads(self) -> int:
        return self.d_inner // self.headdim


# Mamba-2 2.7B (public config: d_model 2560, 64 layers, expand 2, d_state 128, headdim 64, 1 group)
MAMBA2_2P7B = Mamba2Dims(d_model=2560, d_inner=5120, n_layers=64)


def mamba2_weights(m2: Mamba2Dims, layer: int = 0, seed: int = 5000) -> dict:
    """Full weights of one Mamba-2 mixer (float64 CPU; nn.Linear [out, in]); packed
    w_in rows [z (E) | x (E) | B (G N) | C (G N) | dt (H)], Mamba-2 init ranges: projections
    U(+-1/sqrt(fan_in)), conv U(+-1/sqrt(K)), dt_bias = softplus^-1(dt0) with dt0 log-uniform in
    [1e-3, 1e-1], A_log = log U[1, 16] (+ jitter), D = 1, norm weight 1 + N(0, 0.1)."""
    g = torch.Generator().manual_seed(seed + layer)
    D, E, N, G, K = m2.d_model, m2.d_inner, m2.d_state, m2.n_groups, m2.d_conv
    H = m2.n_heads
    C = E + 2 * G * N
    w = {"w_in": _u(g, (2 * E + 2 * G * N + H, D), 1.0 / math.sqrt(D)),
         "conv_w": _u(g, (C, K), 1.0 / math.sqrt(K)), "conv_b": _u(g, (C,), 1.0 / math.sqrt(K))}
    lo, hi = math.log(1e-3), math.log(1e-1)
    dt0 = torch.exp(torch.rand((H,), generator=g, dtype=torch.float64) * (hi - lo) + lo)
    w["dt_bias"] = dt0 + torch.log(-torch.expm1(-dt0))
    w["a_log"] = torch.log(1.0 + 15.0 * torch.rand((H,), generator=g, dtype=torch.float64))
    w["d_skip"] = torch.ones((H,), dtype=torch.float64)
    w["norm_w"] = 1.0 + 0.1 * torch.randn((E,), generator=g, dtype=torch.float64)
    w["w_out"] = _u(g, (D, E), 1.0 / math.sqrt(E)) / math.sqrt(2.0 * max(m2.n_layers, 1))
    return w
