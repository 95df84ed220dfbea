"""Quantised all-reduce oracle (TEST INFRASTRUCTURE ONLY).

PAPER.md:352-359 (§4.4) quantises the communicated tensor "to a lower-precision
representation ... for transfer and reduction, and then dequantizing them
back".  The build's reading (north_star; SURVEY.md §8(c) qar_ref, Q6-Q9):

  per rank r, per block b of `block` consecutive elements of a row:
      amax = max |o|                       (exact in fp32)
      s    = fl32(amax / 127)              (IEEE fp32 division, round-nearest-even)
      q    = clamp(rint_even(fl32(o / s)), -127, 127)   (int8, never -128)
      amax == 0  ->  s = 0, q = 0
  result = sum_{r=0..k-1} s_r * q_r        (fixed rank order)
  bound  |result - sum_r o_r| <= sum_r s_r / 2 <= k * max_r amax_r / 254

Codes and scales are integer/byte results decided in fp32 on both sides, so the
GPU must reproduce them bit-for-bit.  The dequantised sum is formed here in
float64 (each s*q is exact in float64).
"""
from __future__ import annotations

import numpy as np


def quantize_blocks(o, block):
    """o: float32 array [..., n] with n % block == 0.
    Returns (q int8 [..., n], s float32 [..., n // block])."""
    o = np.asarray(o, dtype=np.float32)
    n = o.shape[-1]
    assert n % block == 0, "block must divide the row length (Q7)"
    ob = o.reshape(o.shape[:-1] + (n // block, block))
    amax = np.max(np.abs(ob), axis=-1)                                   # fp32, exact
    s = (amax / np.float32(127.0)).astype(np.float32)                    # fp32 IEEE division
    safe = np.where(s == 0, np.float32(1.0), s).astype(np.float32)
    ratio = (ob / safe[..., None]).astype(np.float32)                    # fp32 IEEE division
    q = np.clip(np.rint(ratio), -127, 127)                               # rint = half-to-even
    q = np.where(s[..., None] == 0, 0, q).astype(np.int8)
    return q.reshape(o.shape), s


def dequantize_blocks(q, s, block):
    """s * q in float64 (exact)."""
    q = np.asarray(q, dtype=np.float64)
    n = q.shape[-1]
    qb = q.reshape(q.shape[:-1] + (n // block, block))
    return (qb * np.asarray(s, dtype=np.float64)[..., None]).reshape(q.shape)


def qallreduce(partials, block):
    """partials: sequence of k float32 arrays (one per rank, same shape).
    Returns (result float64, codes list, scales list)."""
    codes, scales = [], []
    acc = None
    for o in partials:                      # fixed rank order 0..k-1 (Q12)
        q, s = quantize_blocks(o, block)
        codes.append(q)
        scales.append(s)
        d = dequantize_blocks(q, s, block)
        acc = d if acc is None else acc + d
    return acc, codes, scales


def error_bound(scales, block):
    """Per-element bound sum_r s_r / 2 (exact rounding bound of the scheme)."""
    tot = np.sum([np.asarray(s, dtype=np.float64) for s in scales], axis=0) / 2.0
    return np.repeat(tot, block, axis=-1)


def northstar_bound(partials, block):
    """k * max_r amax_{r,b} / 254 per element (north_star closed-form bound)."""
    k = len(partials)
    amaxes = []
    for o in partials:
        o = np.asarray(o, dtype=np.float64)
        n = o.shape[-1]
        amaxes.append(np.max(np.abs(o.reshape(o.shape[:-1] + (n // block, block))), axis=-1))
    m = np.max(np.stack(amaxes), axis=0)
    return np.repeat(k * m / 254.0, block, axis=-1)


# ---------------------------------------------------------------------------------------------
# FP16-wire all-reduce: the paper's own quantisation (§4.4, "quantizing the
# communicated tensors to a lower-precision representation (FP16, from FP32) for transfer and
# reduction, and then dequantizing them back"; "we quantize from the default FP32
# precision to FP16").  Readings (Q21): the cast is IEEE round-to-nearest-even
# (overflow -> inf, as the cast defines); the one-shot schedule reduces the k fp16 values in
# fp32, fixed rank order 0..k-1 (acc = fl32(h_0); acc = fl32(acc + fl32(h_r))), and the fp32
# sum is added to the fp32 residual (Q9).  Every step is an IEEE-defined operation, so the GPU
# must reproduce it bit for bit.

def fp16_cast(o):
    """fl16(o) with round-to-nearest-even (numpy's float32 -> float16 cast)."""
    return np.asarray(o, dtype=np.float32).astype(np.float16)


def fp16_allreduce(partials):
    """partials: k float32 arrays.  Returns the float32 sum of the fp16-cast partials formed
    left to right in fp32 (fixed rank order), and the fp16 wire arrays."""
    wire = [fp16_cast(o) for o in partials]
    acc = wire[0].astype(np.float32)
    for h in wire[1:]:
        acc = (acc + h.astype(np.float32)).astype(np.float32)
    return acc, wire


def fp16_error_bound(partials):
    """Per element: sum_r (|o_r| 2^-11 + 2^-25) (cast error: half an fp16 ulp, relative 2^-11
    in the normal range, absolute 2^-25 in the subnormal range) + the fp32 additions
    ((k-1) roundings of at most 2^-24 |partial sum| each, bounded via sum_r |o_r| (1 + 2^-11))."""
    a = np.sum([np.abs(np.asarray(o, dtype=np.float64)) for o in partials], axis=0)
    k = len(partials)
    cast = a * 2.0 ** -11 + k * 2.0 ** -25
    adds = (k - 1) * 2.0 ** -24 * (a * (1 + 2.0 ** -11) + k * 2.0 ** -25)
    return cast + adds


# ---------------------------------------------------------------------------------------------
# bf16-wire all-reduce: the custom bf16 arm of SURVEY.md §8(d) ("AR#2 in {NCCL bf16, custom bf16,
# int8}"), the unquantised 16-bit baseline the paper's Table 1 compares quantisation against
# (PAPER.md:591-610).  Same one-shot schedule and fp32 reduction as the fp16 wire; the cast is
# bfloat16 round-to-nearest-even (8 significant bits, fp32's exponent range, so no overflow for
# finite fp32 inputs except the last binade rounding up to inf).

def bf16_cast(o):
    """fl_bf16(o), RNE, returned as the float32 values (bfloat16 = the top 16 bits of binary32):
    add 0x7FFF plus the lowest kept bit to the 32-bit pattern, then clear the low 16 bits."""
    u = np.asarray(o, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def bf16_allreduce(partials):
    """partials: k float32 arrays.  Returns the float32 sum of the bf16-cast partials formed left
    to right in fp32 (fixed rank order), and the bf16 wire values (as float32)."""
    wire = [bf16_cast(o) for o in partials]
    acc = wire[0].astype(np.float32)
    for h in wire[1:]:
        acc = (acc + h).astype(np.float32)
    return acc, wire


def bf16_error_bound(partials):
    """Per element: sum_r |o_r| 2^-8 (RNE cast: half a bf16 ulp; 8 significant bits, so the unit
    roundoff is 2^-8; the fp32 subnormal range is ignored) + (k-1) roundings of the fp32 adds,
    each <= 2^-24 sum_r |o_r| (1 + 2^-8)."""
    a = np.sum([np.abs(np.asarray(o, dtype=np.float64)) for o in partials], axis=0)
    k = len(partials)
    return a * 2.0 ** -8 + (k - 1) * 2.0 ** -24 * a * (1 + 2.0 ** -8)


# ---------------------------------------------------------------------------------------------
# Two-shot int8 schedule with SHARED per-block scales (DESIGN.md §3 Q6):
#   A_b   = max_r amax_{r,b}                   (exact in fp32)
#   s_b   = fl32(A_b / 127)                     (IEEE fp32 division)
#   q_r   = clamp(rint_even(fl32(o_r / s_b)), -127, 127)   (0 when s_b = 0)
#   Q     = sum_r q_r                           (exact integer, |Q| <= 127 k: int16 on the wire)
#   out   = fl32(s_b * Q)
# bound |out - sum_r o_r| <= k s_b / 2 (+ the final fp32 rounding) <= k A_b / 254: the north_star's
# k * max|x| / 254 with max over ranks.  The reduce-scatter / all-gather split is a data movement
# choice that does not change these values.

def qallreduce_twoshot(partials, block):
    """partials: k float32 arrays [..., n].  Returns (out float32, codes list, scales float32)."""
    ps = [np.asarray(o, dtype=np.float32) for o in partials]
    n = ps[0].shape[-1]
    assert n % block == 0
    shp = ps[0].shape[:-1] + (n // block, block)
    A = np.max(np.stack([np.max(np.abs(o.reshape(shp)), axis=-1) for o in ps]), axis=0)
    s = (A / np.float32(127.0)).astype(np.float32)
    safe = np.where(s == 0, np.float32(1.0), s).astype(np.float32)
    codes = []
    Q = np.zeros(shp, dtype=np.int64)
    for o in ps:                                   # rank order irrelevant: integer sum
        q = np.clip(np.rint((o.reshape(shp) / safe[..., None]).astype(np.float32)), -127, 127)
        q = np.where(s[..., None] == 0, 0, q).astype(np.int64)
        codes.append(q.reshape(ps[0].shape).astype(np.int8))
        Q += q
    out = (s[..., None] * Q.astype(np.float32)).astype(np.float32)
    return out.reshape(ps[0].shape), codes, s


# ---------------------------------------------------------------------------------------------
# Requantised two-shot int8 schedule (a LABELLED variant, never the default):
# every rank quantises its partial with its own per-block scales (as the one-shot scheme), the
# owner of shard j dequantises and sums the k ranks' codes of its shard in fixed rank order in
# fp32, RE-quantises that sum with a fresh per-block scale, and the requantised shard is all-gathered:
#   S    = fl32(...fl32(fl32(s_0 q_0) + fl32(s_1 q_1)) ... + fl32(s_{k-1} q_{k-1}))
#   q', s' = quantize_blocks(S);   out = fl32(s' q')
# Wire per rank 2 (k-1)/k n (1 + 4/blk) B (k = 4: 1.55 n, k = 8: 1.80 n) at the price of a second
# rounding: |out - sum_r o_r| <= sum_r s_r / 2 + s'/2 <= 2 k max_r amax_r / 254.

def qallreduce_requant(partials, block):
    """partials: k float32 arrays [..., n].  Returns (out float32, first-stage codes/scales lists,
    requantised codes, requantised scales)."""
    codes, scales, S = [], [], None
    for o in partials:
        q, s = quantize_blocks(np.asarray(o, dtype=np.float32), block)
        codes.append(q)
        scales.append(s)
        d = (np.repeat(s, block, axis=-1) * q.astype(np.float32)).astype(np.float32)
        S = d if S is None else (S + d).astype(np.float32)
    q2, s2 = quantize_blocks(S, block)
    out = (np.repeat(s2, block, axis=-1) * q2.astype(np.float32)).astype(np.float32)
    return out, codes, scales, q2, s2
