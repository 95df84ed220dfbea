// gemm_tcgen05.cu — persistent warp-specialised bf16 GEMM for sm_100a.
//
// C = A B^T, A [M,K] and B [N,K] K-major bf16 (activations x nn.Linear weights),
// fp32 accumulation in TMEM.  Used for the token-wise projections of the mixer
// ("token-wise matrix multiplications"): in_proj, x_proj, dt_proj,
// out_proj.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0  : TMA producer — cp.async.bulk.tensor 2D loads of A (128 x 64) and
//             B (BN x 64) tiles, SWIZZLE_128B, into a 4-stage smem ring (mbarrier full/empty)
//   warp 1  : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16 per
//             instruction), commits to the smem-empty barriers and the TMEM-full barrier
//   warps 2-5: epilogue — tcgen05.ld 32x32b.x32 TMEM -> registers, fused epilogue op
//             (bf16 store / fp32 store / softplus(+bias) / fp32 add / fp32 atomic add),
//             optionally transposed for swap-AB decode GEMMs.
// TMEM holds two 256-column accumulators so the epilogue of tile i overlaps the MMAs
// of tile i+1.  Split-K (ksplit > 1) requires the atomic epilogue.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "internal.h"


namespace ssm {

namespace {
constexpr int BM = 128, BK = 64, BN_MAX = 256, MAX_STAGES = 16;
constexpr int A_STAGE = BM * BK * 2;      // 16 KB
constexpr int SMEM_BYTES = 227 * 1024;              // ring stages are sized to fill what is left
constexpr int RING_BYTES = SMEM_BYTES - 1024 - 512;
// stage = A tile (128 x 64 bf16) + B tile (BN x 64 bf16); as many stages as fit (small-N decode
// GEMMs are latency-bound weight streams and need many bytes in flight)
// A stage holds KBS consecutive 64-wide k-blocks of A and B: [KBS x A tile][KBS x B tile].
__host__ __device__ inline int stage_bytes(int BN, int KBS) { return KBS * (A_STAGE + BN * BK * 2); }
__host__ __device__ inline int num_stages(int BN, int KBS, int ring = RING_BYTES) {
  const int s = ring / stage_bytes(BN, KBS);
  return s > MAX_STAGES ? MAX_STAGES : s;
}
// Per-launch shape of the CTA's resources: smem ring size and TMEM accumulator columns (two
// accumulators of acc_stride columns).  Smaller values let two CTAs share an SM.
struct CtaRes {
  int ring;          // bytes of the stage ring
  int tmem_cols;     // power of two >= 32
  int acc_stride;    // columns per accumulator
  int a_indep;       // A (weights) does not depend on the predecessor grid: first ring fill before the PDL wait
};
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (2 per TMEM lane group)
// threads of a kernel variant: the skinny atomic variant (VAR 2, BN <= 32: one 32-column chunk, so
// only the first epilogue half ever works) runs 4 epilogue warps -- a smaller CTA that fits next
// to the decode-step blocks it follows
constexpr int var_threads(int var) { return var == 2 ? 192 : kThreads; }
// VAR 6: the prefill dt_proj with its softplus(+bias) epilogue fixed at compile time; VAR 7: the
// prefill out_proj with the int8 quantisation epilogue (EPI_QUANT_I8)
constexpr int var_kind(int var) { return var == 6 ? EPI_SOFTPLUS_BF16 : var == 7 ? EPI_QUANT_I8 : -1; }

// Work decomposition: unit u = (k-split, m-tile, n-tile), CTAs stride over units.
struct TileSched {
  int m_tiles, n_tiles, kb_total, kbs, ksplit, units;
  int grp;  // CTAs per unit: 1, or 2 for a CTA pair (cta_group::2) sharing one M = 256 tile
  // iterate units (mt, nt, kb0, kb1) of this CTA; returns false when done
  __device__ bool next(int& cursor, int& mt, int& nt, int& kb0, int& kb1) const {
    const int u = cursor;
    if (u >= units) return false;
    cursor += gridDim.x / grp;
    nt = u % n_tiles;
    const int rest = u / n_tiles;
    mt = rest % m_tiles;
    const int ks = rest / m_tiles;
    kb0 = ks * kbs;
    kb1 = min(kb_total, kb0 + kbs);
    return true;
  }
  __device__ int first() const { return (int)blockIdx.x / grp; }
};

// Optional row scale 1 / sqrt(rss[r] * rss_inv + rss_eps) of logical row r (Epilogue::rss).
__device__ __forceinline__ float rss_scale(const Epilogue& e, int r) { return rsqrtf(e.rss[r] * e.rss_inv + e.rss_eps); }
// trans = 1: the logical rows are the 32 columns n0..n0+31 of the chunk
__device__ __forceinline__ void rss_apply_trans(const Epilogue& e, int n0, int N, float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (n0 + j < N) v[j] *= rss_scale(e, n0 + j);
}

// The only epilogue of the VAR 2 kernel: C[n * ldc + m] += acc atomically (swap-AB split-K).
__device__ __forceinline__ void epi_chunk_atomic_trans(const Epilogue& e, int m0, int n0, int M, int N,
                                                       uint32_t (&r)[32]) {
  const int m = m0 + threadIdx.x % 32;
  if (m >= M) return;
  const int nv = min(32, N - n0);
  float* C = reinterpret_cast<float*>(e.C) + (int64_t)n0 * e.ldc + m;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (e.rss) rss_apply_trans(e, n0, N, v);
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j < nv) atomicAdd(C + (int64_t)j * e.ldc, v[j]);
}

// Epilogue for one warp's 32 x 32 chunk: lane = row m0 + lane, columns n0..n0+31, stored
// straight from registers (staging through shared memory would compete with the UMMA operand
// reads for smem bandwidth in the MMA-bound projections).
template <int FK = -1>  // FK >= 0: the epilogue kind is fixed at compile time (other paths pruned)
__device__ __forceinline__ void epi_chunk(const Epilogue& e, int m0, int n0, int M, int N, uint32_t (&r)[32],
                                          const float* bpre = nullptr) {
  const int kind = FK >= 0 ? FK : e.kind;
  const int m = m0 + threadIdx.x % 32;
  if (m >= M) return;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (kind == EPI_SOFTPLUS_BF16 || kind == EPI_SOFTPLUS_F32) {
    float bb[32];
    if (bpre) {  // bias chunk loaded by the caller before the TMEM load (latencies overlap)
#pragma unroll
      for (int j = 0; j < 32; ++j) bb[j] = bpre[j];
    } else if (e.trans) {
      const float b0 = e.bias[m];
#pragma unroll
      for (int j = 0; j < 32; ++j) bb[j] = b0;
    } else if (n0 + 32 <= N && ((reinterpret_cast<uintptr_t>(e.bias + n0) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // 8 broadcast 16-B loads, all issued before use
        const float4 t4 = reinterpret_cast<const float4*>(e.bias + n0)[q];
        bb[4 * q] = t4.x; bb[4 * q + 1] = t4.y; bb[4 * q + 2] = t4.z; bb[4 * q + 3] = t4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) bb[j] = (n0 + j < N) ? e.bias[n0 + j] : 0.f;
    }
    if (kind == EPI_SOFTPLUS_BF16) {  // bf16 output: one-MUFU softplus (error far below bf16 rounding)
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = softplus_1mufu(v[j] + bb[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = softplus(v[j] + bb[j]);
    }
  }
  if (FK < 0 && e.rss) {
    if (e.trans) {
      rss_apply_trans(e, n0, N, v);
    } else {
      const float sc = rss_scale(e, m);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= sc;
    }
  }
  if (e.trans) {
    // element (m, n) -> C[n * ldc + m]; lanes hold consecutive m -> coalesced per n.  One loop per
    // kind (no per-element dispatch), valid columns first so all stores issue back to back.
    const int nv = min(32, N - n0);
    if (kind == EPI_STORE_BF16 || kind == EPI_SOFTPLUS_BF16) {
      __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(e.C) + (int64_t)n0 * e.ldc + m;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nv) C[(int64_t)j * e.ldc] = __float2bfloat16_rn(v[j]);
    } else if (kind == EPI_STORE_F32 || kind == EPI_SOFTPLUS_F32) {
      float* C = reinterpret_cast<float*>(e.C) + (int64_t)n0 * e.ldc + m;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nv) C[(int64_t)j * e.ldc] = v[j];
    } else if (kind == EPI_ADD_F32) {
      float* C = reinterpret_cast<float*>(e.C) + (int64_t)n0 * e.ldc + m;
      float o[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nv) o[j] = C[(int64_t)j * e.ldc];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nv) C[(int64_t)j * e.ldc] = o[j] + v[j];
    } else {
      float* C = reinterpret_cast<float*>(e.C) + (int64_t)n0 * e.ldc + m;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nv) atomicAdd(C + (int64_t)j * e.ldc, v[j]);
    }
    return;
  }
  if (FK < 0 && kind == EPI_SPLIT_DBC) {  // the chunk lies in one field of one head (R, P multiples of 32)
    const int hd = n0 / e.dbc_P, c = n0 % e.dbc_P;
    if (c < e.dbc_R) {
      uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.dbc_low) +
                                           ((int64_t)hd * e.dbc_M + m) * e.dbc_R + c);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __nv_bfloat162 t2 = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
          pw[j] = *reinterpret_cast<uint32_t*>(&t2);
        }
        d4[q] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
      }
    } else {
      float4* d4 = reinterpret_cast<float4*>(e.dbc_bc + ((int64_t)hd * e.dbc_M + m) * (e.dbc_P - e.dbc_R) + c - e.dbc_R);
#pragma unroll
      for (int q = 0; q < 8; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    return;
  }
  const bool full = (n0 + 32 <= N);
  const int64_t base = (int64_t)m * e.ldc + n0;
  if (kind == EPI_STORE_BF16 || kind == EPI_SOFTPLUS_BF16) {
    __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(e.C) + base;
    if (full && ((reinterpret_cast<uintptr_t>(C) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 pk;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __nv_bfloat162 t2 = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
          pw[j] = *reinterpret_cast<uint32_t*>(&t2);
        }
        reinterpret_cast<uint4*>(C)[q] = pk;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) C[j] = __float2bfloat16_rn(v[j]);
    }
    return;
  }
  float* C = reinterpret_cast<float*>(e.C) + base;
  const bool vec = full && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  if (kind == EPI_STORE_F32 || kind == EPI_SOFTPLUS_F32) {
    if (vec) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(C)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) C[j] = v[j];
    }
  } else if (kind == EPI_ADD_F32) {
    if (vec) {
      float4 o[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = reinterpret_cast<const float4*>(C)[q];   // all loads first
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        o[q].x += v[4 * q]; o[q].y += v[4 * q + 1]; o[q].z += v[4 * q + 2]; o[q].w += v[4 * q + 3];
        reinterpret_cast<float4*>(C)[q] = o[q];
      }
      if (FK < 0 && e.cpy) {  // bf16 copy of the updated rows + their sums of squares (Epilogue::cpy / ssq)
        uint4* cp = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.cpy) + base);
        float sq = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 a = o[2 * q], b = o[2 * q + 1];
          sq = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, sq))));
          sq = fmaf(b.x, b.x, fmaf(b.y, b.y, fmaf(b.z, b.z, fmaf(b.w, b.w, sq))));
          __nv_bfloat162 t0 = __floats2bfloat162_rn(a.x, a.y), t1 = __floats2bfloat162_rn(a.z, a.w);
          __nv_bfloat162 t2 = __floats2bfloat162_rn(b.x, b.y), t3 = __floats2bfloat162_rn(b.z, b.w);
          cp[q] = make_uint4(*reinterpret_cast<uint32_t*>(&t0), *reinterpret_cast<uint32_t*>(&t1),
                             *reinterpret_cast<uint32_t*>(&t2), *reinterpret_cast<uint32_t*>(&t3));
        }
        e.ssq[(int64_t)m * ((N + 31) / 32) + n0 / 32] = sq;
      }
    } else {
      float sq = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) {
          const float o = C[j] + v[j];
          C[j] = o;
          if (FK < 0 && e.cpy) {
            reinterpret_cast<__nv_bfloat16*>(e.cpy)[base + j] = __float2bfloat16_rn(o);
            sq = fmaf(o, o, sq);
          }
        }
      if (FK < 0 && e.cpy) e.ssq[(int64_t)m * ((N + 31) / 32) + n0 / 32] = sq;
    }
  } else {  // EPI_ATOMIC_F32
    if (vec) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        atomicAdd(reinterpret_cast<float4*>(C) + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) atomicAdd(C + j, v[j]);
    }
  }
}

// ---- EPI_QUANT_I8: int8 per-block quantisation of the out_proj partial in its TMEM drain -------
// (§4.4; reading Q6-Q8.)  The tile's rows are the TMEM lanes, a
// row's qblk-column block spans qblk / 32 chunks of 32 columns that the two epilogue halves drain
// alternately, so the drain runs twice: pass 1 writes each chunk's amax to shared memory
// (s_am [128 rows][8 chunks]), pass 2 re-reads the accumulator, forms s = fl32(amax / 127) of the
// chunk's block and stores the 32 codes (two 16-B stores) -- the same IEEE operations as
// quantize_kernel, so codes and scales equal the fp32-partial route bit for bit.
__device__ __forceinline__ void quant_epilogue(const Epilogue& e, int m0, int n_base, int BN, int M, int N,
                                               uint32_t tbase, float* s_am) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = (warp - 2) >> 2, eg = warp & 3;
  const int row = eg * 32 + lane, m = m0 + lane;
  const int nch = BN / 32, cpb = e.qblk / 32;
  const float rsc = (e.rss && m < M) ? rss_scale(e, m) : 1.f;  // row scale applied before quantising
  for (int c = half; c < nch; c += 2) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tbase + c * 32, r);
    tmem_ld_wait();
    float am = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) am = fmaxf(am, fabsf(__uint_as_float(r[j]) * rsc));
    s_am[row * 8 + c] = am;
  }
  named_bar_sync(1, 256);
  for (int c = half; c < nch; c += 2) {
    const int n0 = n_base + c * 32;
    const int b0 = (c / cpb) * cpb;
    float A = 0.f;
    for (int j = 0; j < cpb; ++j) A = fmaxf(A, s_am[row * 8 + b0 + j]);
    const float s = __fdiv_rn(A, 127.0f);
    uint32_t r[32];
    tmem_ld_32x32b_x32(tbase + c * 32, r);
    tmem_ld_wait();
    if (m < M && n0 < N) {
      uint32_t pk[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int code = 0;
          if (s != 0.f) code = max(-127, min(127, __float2int_rn(__fdiv_rn(__uint_as_float(r[4 * q + j]) * rsc, s))));
          w |= (uint32_t)(code & 0xff) << (8 * j);
        }
        pk[q] = w;
      }
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(e.C) + (int64_t)m * e.ldc + n0);
      dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      if (c % cpb == 0) e.qs[(int64_t)m * (N / e.qblk) + n0 / e.qblk] = s;
    }
  }
  named_bar_sync(1, 256);  // s_am reused by the next tile
}

// ---- EPI_DECODE_INPROJ: decode in_proj epilogue fused with the conv step and x_proj ----------
// Epilogue warp w (0..7) owns TMEM lane group eg = w % 4 (feature rows f0 + 32 eg + lane) and the
// batch columns [16 half, 16 half + 16) (half = w / 4), so a CTA covers N <= 32 decode tokens.
constexpr int SU_LD = 136;                       // u tile row pitch (bf16): conflict-free ldmatrix
constexpr int SU_BYTES = 32 * SU_LD * 2;         // u tile [32 tokens][128 channels] bf16
constexpr int XP_NT = 5;                         // x_proj n-tiles (8 outputs) per warp: P <= 320 (Zamba: 264)

template <int XPN = XP_NT>  // x_proj n-tiles per warp: P <= 64 XPN
__device__ __forceinline__ void decode_inproj_epilogue(const Epilogue& e, const TileSched& ts, int M, int N,
                                                       uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base,
                                                       const CtaRes& cr, __nv_bfloat16* su) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int eg = warp & 3, half = (warp - 2) >> 2, ew = warp - 2;
  const int Ek = e.Ek, K = e.K, P = e.P, ldx = e.hl * e.P;
  __nv_bfloat16* cst = reinterpret_cast<__nv_bfloat16*>(e.cst);
  const __nv_bfloat16* wx = reinterpret_cast<const __nv_bfloat16*>(e.wx);
  int acc = 0;
  uint32_t acc_ph = 0;
  int cur = ts.first(), mt, nt, kb0, kb1;
  while (ts.next(cur, mt, nt, kb0, kb1)) {
    if (kb0 >= kb1) continue;
    const int f0 = mt * BM;
    const int f = f0 + eg * 32 + lane;
    const bool is_x = f < Ek;
    const bool tile_x = f0 < Ek;
    // ---- loads that do not depend on the GEMM, issued while the weight stream is in flight
    float wv[4] = {0.f, 0.f, 0.f, 0.f}, bias = 0.f;
    uint32_t win[3][8];  // cached window, bf16 pairs (tokens 2i, 2i+1 of this warp's 16)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int q = 0; q < 8; ++q) win[j][q] = 0u;
    if (is_x) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < K) wv[j] = e.cw[(int64_t)f * K + j];
      bias = e.cb[f];
      const uint16_t* cs16 = reinterpret_cast<const uint16_t*>(cst);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int b = half * 16 + q;
        if (b < N)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (j < K - 1) win[j][q / 2] |= (uint32_t)cs16[((int64_t)b * (K - 1) + j) * Ek + f] << (16 * (q & 1));
      }
    }
    uint32_t wf[XPN][8][2];  // W_x B-fragments: rows p = 8 nt + lane / 4, cols f0 + 16 ks + 2 (lane % 4) (+8)
    const int hd = f0 / e.cph;
    if (tile_x) {
#pragma unroll
      for (int i = 0; i < XPN; ++i) {
        const int p = (ew + 8 * i) * 8 + lane / 4;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const int fc = f0 + ks * 16 + 2 * (lane & 3);
          const __nv_bfloat16* row = wx + (int64_t)(hd * P + p) * Ek;
          wf[i][ks][0] = (p < P && fc < Ek) ? *reinterpret_cast<const uint32_t*>(row + fc) : 0u;
          wf[i][ks][1] = (p < P && fc + 8 < Ek) ? *reinterpret_cast<const uint32_t*>(row + fc + 8) : 0u;
        }
      }
    }
    // ---- accumulator: 16 token columns of this warp's 32 feature rows
    mbar_wait(&tfull[acc], acc_ph);
    tc_fence_after();
    uint32_t r[16];
    const uint32_t tb = tmem_base + ((uint32_t)(eg * 32) << 16) + (uint32_t)(acc * cr.acc_stride + half * 16);
    tmem_ld_32x32b_x16(tb, r);
    tmem_ld_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[acc]);  // TMEM consumed: the MMA warp may reuse it
    if (++acc == 2) { acc = 0; acc_ph ^= 1; }

    __nv_bfloat16* su_col = su + (f - f0);
    if (is_x) {
      // causal conv step (tap K-1 = current token) + SiLU; window shift
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int b = half * 16 + q;
        float uq = 0.f;
        if (b < N) {
          const float x = __bfloat162float(__float2bfloat16_rn(__uint_as_float(r[q])));
          float a = bias;
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (j < K - 1) a = fmaf(wv[j], __uint_as_float((win[j][q / 2] >> (16 * (q & 1))) << 16), a);
          float wl = wv[1];
#pragma unroll
          for (int j = 2; j < 4; ++j)
            if (j == K - 1) wl = wv[j];
          a = fmaf(wl, x, a);
          const __nv_bfloat16 ub = __float2bfloat16_rn(silu<true>(a));
          reinterpret_cast<__nv_bfloat16*>(e.u)[(int64_t)b * Ek + f] = ub;
          uq = __bfloat162float(ub);
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (j < K - 2)
              reinterpret_cast<uint16_t*>(cst)[((int64_t)b * (K - 1) + j) * Ek + f] =
                  (uint16_t)(win[j + 1][q / 2] >> (16 * (q & 1)));
          cst[((int64_t)b * (K - 1) + (K - 2)) * Ek + f] = __float2bfloat16_rn(x);
        }
        su_col[b * SU_LD] = __float2bfloat16_rn(uq);
      }
    } else {
      if (f < M) {
        __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(e.C) + f;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int b = half * 16 + q;
          if (b < N) C[(int64_t)b * e.ldc] = __float2bfloat16_rn(__uint_as_float(r[q]));
        }
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) su_col[(half * 16 + q) * SU_LD] = __float2bfloat16_rn(0.f);
    }
    named_bar_sync(1, 256);
    if (tile_x) {
      // x_proj partial of this tile's 128 channels: xacc[b][hd P + p] += sum_f u[b][f] W_x[hd P + p][f]
      for (int mi = 0; mi * 16 < N; ++mi) {
        uint32_t a[8][4];
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          ldmatrix_x4(a[ks], su + (mi * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * SU_LD + ks * 16 + (lane >> 4) * 8);
#pragma unroll
        for (int i = 0; i < XPN; ++i) {
          const int p0 = (ew + 8 * i) * 8;
          if (p0 >= P) continue;
          float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) mma_16816_bf16(d, a[ks], wf[i][ks][0], wf[i][ks][1]);
          const int p = p0 + 2 * (lane & 3);
          const int b = mi * 16 + lane / 4;
          if (p < P) {
            if (b < N) red_add_v2(e.xacc + (int64_t)b * ldx + hd * P + p, d[0], d[1]);
            if (b + 8 < N) red_add_v2(e.xacc + (int64_t)(b + 8) * ldx + hd * P + p, d[2], d[3]);
          }
        }
      }
    }
    named_bar_sync(1, 256);  // u tile free for the next tile
  }
}

// Epilogue warp done with an accumulator: a pair's MMA issuer (the leader) waits for both CTAs.
template <int CG>
__device__ __forceinline__ void tempty_arrive(uint64_t* bar) {
  if constexpr (CG == 2) mbar_arrive_remote(mapa_shared(bar, 0));
  else mbar_arrive(bar);
}

// VAR: 0 = every path (prefill GEMMs); 1 = the fused decode in_proj only; 2 = skinny swap-AB
// split-K GEMMs with the atomic epilogue only (decode out_proj / x_proj); 6 = prefill dt_proj
// (softplus epilogue).  The decode variants are separate kernels so their register allocation is
// not set by paths they never run.
// CG = 2: CTA pair (2-CTA cluster).  The pair computes a 256 x BN tile with cta_group::2 UMMAs
// issued by the leader (rank 0): each CTA TMA-loads its 128 rows of A and BN / 2 rows of B, both
// halves' transaction bytes complete on the leader's full barrier, the leader's commits arrive on
// both CTAs' empty / TMEM-full barriers (multicast), and each CTA's epilogue drains its own 128
// accumulator lanes, then arrives on the leader's TMEM-empty barrier.  Per CTA and k-block the ring
// takes 32 KB instead of 48 KB for the same MMA work (the B tile is shared): a third less L2 -> SM
// operand traffic, the limit of the 1-CTA kernel on the prefill projections.
template <int VAR, int XPN = XP_NT, int CG = 1>
__global__ void __launch_bounds__(var_threads(VAR), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int BN, int KBS, TileSched ts, Epilogue epi, const __nv_bfloat16* a_blk, int64_t lda, int K,
                   CtaRes cr, int a_blocked) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int BNL = BN / CG;  // B rows this CTA loads
  const int STAGES = num_stages(BNL, KBS, cr.ring);
  const int SB = stage_bytes(BNL, KBS);
  const int BOFF = KBS * A_STAGE;  // B tiles follow the KBS A tiles (1024-B aligned)
  const int BSUB = BNL * BK * 2;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const int row_off = (int)rank * BM;  // this CTA's rows inside the pair's 256-row tile
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + cr.ring);
  uint64_t* empty = full + MAX_STAGES;
  uint64_t* tfull = empty + MAX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    if (!a_blocked) tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CG * (var_threads(VAR) - 64) / 32);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair(tmem_slot, cr.tmem_cols);
    else tmem_alloc(tmem_slot, cr.tmem_cols);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer.  The whole warp runs the (warp-uniform) schedule and waits;
    // lane 0 alone issues the copies.  (With lane 0 looping alone while lanes 1-31 sat at the
    // teardown barrier, every iteration of the producer loop measured ~0.2-0.45 us.)
    const bool leader = lane == 0;
    const uint32_t stage_tx = (uint32_t)CG * (BM + BNL) * BK * 2;  // per k-block (both CTAs of a pair)
    const uint32_t full_remote = CG == 2 ? mapa_shared(full, 0) : 0u;  // leader's full[0]
    auto issue_a = [&](uint8_t* st, uint64_t* bar, int mt, int kb, int nk) {
      if (a_blocked)  // A pre-tiled AND pre-swizzled: the nk blocks (mt, kb..kb+nk) are one
        // contiguous run of nk x 16 KB whose bytes are already the SW128 smem image -> 1D bulk copy
        bulk_load_evict_first(st, a_blk + ((int64_t)mt * ts.kb_total + kb) * (BM * BK), (uint32_t)nk * A_STAGE, bar);
      else if constexpr (CG == 2)
        for (int j = 0; j < nk; ++j)
          tma_load_2d_pair(st + j * A_STAGE, &tmA, full_remote + (uint32_t)((bar - full) * 8), (kb + j) * BK,
                           mt * BM * CG + row_off);
      else
        for (int j = 0; j < nk; ++j) tma_load_2d(st + j * A_STAGE, &tmA, bar, (kb + j) * BK, mt * BM);
    };
    auto issue_b = [&](uint8_t* st, uint64_t* bar, int nt, int kb, int nk) {
      if constexpr (CG == 2)
        for (int j = 0; j < nk; ++j)
          tma_load_2d_pair(st + BOFF + j * BSUB, &tmB, full_remote + (uint32_t)((bar - full) * 8), (kb + j) * BK,
                           nt * BN + (int)rank * BNL);
      else
        for (int j = 0; j < nk; ++j) tma_load_2d(st + BOFF + j * BSUB, &tmB, bar, (kb + j) * BK, nt * BN);
    };
    // A independent of the predecessor grid (weights): arm the first ring fill and issue its A
    // loads BEFORE griddepcontrol.wait, so the weight stream starts while the predecessor drains.
    int n_pre = 0;
    if (CG == 1 && cr.a_indep) {
      int cur = ts.first(), mt, nt, kb0, kb1;
      while (n_pre < STAGES && ts.next(cur, mt, nt, kb0, kb1))
        for (int kb = kb0; kb < kb1 && n_pre < STAGES; kb += KBS, ++n_pre) {
          const int nk = min(KBS, kb1 - kb);
          if (leader) {
            mbar_arrive_expect_tx(&full[n_pre], (uint32_t)nk * stage_tx);
            issue_a(ring + n_pre * SB, &full[n_pre], mt, kb, nk);
          }
        }
    }
    __syncwarp();
    pdl_wait();
    int stage = 0, g = 0;
    uint32_t ph = 0;
    int cur = ts.first(), mt, nt, kb0, kb1;
    while (ts.next(cur, mt, nt, kb0, kb1)) {
      for (int kb = kb0; kb < kb1; kb += KBS, ++g) {
        const int nk = min(KBS, kb1 - kb);
        uint8_t* st = ring + stage * SB;
        if (g >= n_pre) {
          mbar_wait(&empty[stage], ph ^ 1);
          if (leader) {
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], (uint32_t)nk * stage_tx);
            issue_a(st, &full[stage], mt, kb, nk);
          }
        }
        if (leader) issue_b(st, &full[stage], nt, kb, nk);
        __syncwarp();
        if (++stage == STAGES) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    if (CG == 1 || rank == 0) {  // the leader issues the pair's MMAs
      // ---------------- MMA issuer: the whole warp runs the (warp-uniform) schedule so the UMMA
      // descriptors live in uniform registers; one elected lane issues the tcgen05.mma / commits.
      // (A single-lane loop makes ptxas wrap every UMMA in a uniform-broadcast waterfall loop,
      // ~100 cycles per instruction: that, not the tensor pipe, bounded skinny weight streams.)
      const uint32_t idesc = umma_idesc_bf16(BM * CG, BN);
      const uint64_t ring_desc = umma_desc_sw128(smem_u32(ring));  // + (byte offset >> 4) addresses inside the ring
      int stage = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      int cur = ts.first(), mt, nt, kb0, kb1;
      while (ts.next(cur, mt, nt, kb0, kb1)) {
        if (kb0 >= kb1) continue;
        mbar_wait(&tempty[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * cr.acc_stride);
        for (int kb = kb0; kb < kb1; kb += KBS) {
          const int nk = min(KBS, kb1 - kb);
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          const uint64_t a_desc = ring_desc + (uint64_t)((stage * SB) >> 4);
          const uint64_t b_desc = a_desc + (uint64_t)(BOFF >> 4);
          if (elect_one()) {
            for (int j = 0; j < nk; ++j) {
  #pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = a_desc + (uint64_t)((j * A_STAGE + k * 32) >> 4);
                const uint64_t bd = b_desc + (uint64_t)((j * BSUB + k * 32) >> 4);
                const uint32_t accum = (kb > kb0 || j > 0 || k > 0) ? 1u : 0u;
                if constexpr (CG == 2) umma_bf16_pair(d, ad, bd, idesc, accum);
                else umma_bf16(d, ad, bd, idesc, accum);
              }
            }
            if constexpr (CG == 2) umma_commit_pair(&empty[stage], 3);
            else umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
        if (elect_one()) {
          if constexpr (CG == 2) umma_commit_pair(&tfull[acc], 3);
          else umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9; TMEM lane group = warp % 4, column half = (warp-2)/4
    pdl_wait();
    if (epi.zero && blockIdx.x == 0) {
      const int64_t n4 = epi.nzero / 4;
      for (int64_t i = threadIdx.x - 64; i < n4; i += var_threads(VAR) - 64)
        reinterpret_cast<float4*>(epi.zero)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t i = 4 * n4 + threadIdx.x - 64; i < epi.nzero; i += var_threads(VAR) - 64) epi.zero[i] = 0.f;
    }
    // VAR 6 (prefill dt_proj): the bias vector staged in shared memory once per CTA, so the epilogue's
    // per-chunk bias reads are LDS instead of global loads on the drain's critical path (ncu: the
    // dominant stall of this kernel)
    float* sbias = reinterpret_cast<float*>(smem + cr.ring + 512);
    if constexpr (VAR == 6) {
      if (epi.bias)
        for (int i = threadIdx.x - 64; i < N; i += var_threads(VAR) - 64) sbias[i] = epi.bias[i];
      named_bar_sync(1, var_threads(VAR) - 64);
    }
    if constexpr (VAR == 1) {
      decode_inproj_epilogue<XPN>(epi, ts, M, N, tfull, tempty, tmem_base, cr,
                                  reinterpret_cast<__nv_bfloat16*>(smem + cr.ring + 512));
    } else {
      const int eg = warp & 3;
      const int half = (warp - 2) >> 2;
      int acc = 0;
      uint32_t acc_ph = 0;
      int cur = ts.first(), mt, nt, kb0, kb1;
      if (lane == 0) {
        // Touch the first output address now: a TLB miss on a store would otherwise stall the
        // epilogue for microseconds after the weight stream (page walks queue behind it).
        int c2 = cur, mt2, nt2, k0, k1;
        if (ts.next(c2, mt2, nt2, k0, k1)) {
          const int m = min(M - 1, mt2 * BM * CG + row_off + eg * 32), n = min(N - 1, nt2 * BN);
          const int64_t idx = epi.trans ? (int64_t)n * epi.ldc + m : (int64_t)m * epi.ldc + n;
          const int esz = (epi.kind == EPI_STORE_BF16 || epi.kind == EPI_SOFTPLUS_BF16) ? 2 : 4;
          touch_global(reinterpret_cast<const uint8_t*>(epi.C) + idx * esz);
          if (epi.bias) touch_global(epi.bias + (epi.trans ? m : n));
        }
      }
      while (ts.next(cur, mt, nt, kb0, kb1)) {
        if (kb0 >= kb1) continue;
        mbar_wait(&tfull[acc], acc_ph);
        tc_fence_after();
        const int m0 = mt * BM * CG + row_off + eg * 32;
        const uint32_t tbase = tmem_base + ((uint32_t)(eg * 32) << 16) + (uint32_t)(acc * cr.acc_stride);
        if constexpr (VAR == 7) {
          quant_epilogue(epi, m0, nt * BN, BN, M, N, tbase, reinterpret_cast<float*>(smem + cr.ring + 512));
          tc_fence_before();
          __syncwarp();
          if (lane == 0) tempty_arrive<CG>(&tempty[acc]);
          if (++acc == 2) { acc = 0; acc_ph ^= 1; }
          continue;
        }
        if constexpr (VAR == 6) {
          // dt_proj: the warp drains 64 consecutive columns (chunk pairs 2 half + 4 i, + 1) of its 32 rows,
          // softplus(+bias) in registers, bf16 rows staged in shared memory (144-B pitch: conflict-free),
          // then written back as full 128-B row segments (8 lanes per row, 4 rows per store instruction)
          // instead of 32 rows x 16 B per store (measured: the row-per-lane stores were 140 of 336 us)
          uint8_t* stg = smem + cr.ring + 512 + ((N * 4 + 127) / 128 * 128) + (warp - 2) * (32 * 144);
          const int nlim = min(N, nt * BN + BN);  // (an odd chunk count leaves the last pair half empty)
          for (int cp = 2 * half; cp < (BN + 31) / 32; cp += 4) {
            const int n0 = nt * BN + cp * 32;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              uint32_t r[32];
              const int nc = n0 + k * 32;
              float bb[32];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 t4 = (epi.bias && nc + 32 <= N) ? reinterpret_cast<const float4*>(sbias + nc)[q]
                                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                bb[4 * q] = t4.x; bb[4 * q + 1] = t4.y; bb[4 * q + 2] = t4.z; bb[4 * q + 3] = t4.w;
              }
              tmem_ld_32x32b_x32(tbase + (cp + k) * 32, r);
              tmem_ld_wait();
              uint32_t pk[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                float y[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  y[h] = softplus_1mufu(__uint_as_float(r[2 * j + h]) + bb[2 * j + h]);
                }
                __nv_bfloat162 t2 = __floats2bfloat162_rn(y[0], y[1]);
                pk[j] = *reinterpret_cast<uint32_t*>(&t2);
              }
              uint4* dst = reinterpret_cast<uint4*>(stg + lane * 144 + k * 64);
#pragma unroll
              for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int row = it * 4 + (lane >> 3), seg = lane & 7;
              const int m = m0 + row, n = n0 + seg * 8;
              const uint4 v = *reinterpret_cast<const uint4*>(stg + row * 144 + seg * 16);
              if (m < M && n + 8 <= nlim)
                *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(epi.C) + (int64_t)m * epi.ldc + n) = v;
              else if (m < M)
                for (int j = 0; j < 8 && n + j < nlim; ++j)
                  reinterpret_cast<__nv_bfloat16*>(epi.C)[(int64_t)m * epi.ldc + n + j] =
                      reinterpret_cast<const __nv_bfloat16*>(&v)[j];
            }
            __syncwarp();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) tempty_arrive<CG>(&tempty[acc]);
          if (++acc == 2) { acc = 0; acc_ph ^= 1; }
          continue;
        }
        for (int c = half; c < (BN + 31) / 32; c += 2) {
          uint32_t r[32];
          const int nc = nt * BN + c * 32;
          float bpre[32];
          const bool pre = (VAR == 0 || VAR == 6) && (epi.kind == EPI_SOFTPLUS_BF16 || epi.kind == EPI_SOFTPLUS_F32) &&
                           !epi.trans && nc + 32 <= N && ((reinterpret_cast<uintptr_t>(epi.bias + nc) & 15) == 0);
          if (pre) {
            const float* bsrc = (VAR == 6 && epi.bias) ? sbias : epi.bias;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 t4 = reinterpret_cast<const float4*>(bsrc + nc)[q];
              bpre[4 * q] = t4.x; bpre[4 * q + 1] = t4.y; bpre[4 * q + 2] = t4.z; bpre[4 * q + 3] = t4.w;
            }
          }
          tmem_ld_32x32b_x32(tbase + c * 32, r);
          tmem_ld_wait();
          if constexpr (VAR == 2) epi_chunk_atomic_trans(epi, m0, nt * BN + c * 32, M, N, r);
          else epi_chunk<var_kind(VAR)>(epi, m0, nt * BN + c * 32, M, N, r, pre ? bpre : nullptr);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) tempty_arrive<CG>(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // the leader's MMAs write the peer's TMEM: free it after both drained
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_pair(tmem_base, cr.tmem_cols);
    else tmem_dealloc(tmem_base, cr.tmem_cols);
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
// Blocked ("pre-tiled") weight layout: block (r / 128, k / 64) of 128 x 64 bf16 stored as one
// contiguous 16 KB tile, blocks ordered row-tile-major, and each tile stored in the SWIZZLE_128B
// byte order UMMA reads from shared memory (16-B chunk j of row r at position j ^ (r % 8)).  A
// weight-streaming decode GEMM then fetches KBS consecutive k-blocks as ONE 1D bulk copy with
// no tensor-map address generation; the smem image is byte-identical to what a swizzling 2D
// TMA load of the row-major matrix would produce.
__global__ void pack_blocked_kernel(const __nv_bfloat16* __restrict__ w, int rows, int cols, int64_t ld,
                                    __nv_bfloat16* __restrict__ out, int kbt, int64_t n_vec) {
  // one thread per 16-B output vector (8 bf16); zero padding beyond rows / cols
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_vec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = v / (BM * BK / 8);
    const int c = (int)(v % (BM * BK / 8));  // 16-B chunk within the tile: row c / 8, slot c % 8
    const int rr = c >> 3;
    const int r = (int)(blk / kbt) * BM + rr;
    const int k = (int)(blk % kbt) * BK + (((c & 7) ^ (rr & 7)) << 3);
    uint4 val = make_uint4(0, 0, 0, 0);
    if (r < rows) {
      if (k + 8 <= cols && ((ld * 2) % 16 == 0)) {
        val = *reinterpret_cast<const uint4*>(w + (int64_t)r * ld + k);
      } else {
        __nv_bfloat16* t = reinterpret_cast<__nv_bfloat16*>(&val);
        for (int j = 0; j < 8; ++j) t[j] = (k + j < cols) ? w[(int64_t)r * ld + k + j] : __float2bfloat16_rn(0.f);
      }
    }
    reinterpret_cast<uint4*>(out)[v] = val;
  }
}
}  // namespace

bool encode_tmap_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int elem_bytes,
                    int box_cols, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc || (elem_bytes != 2 && elem_bytes != 4)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * elem_bytes)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

size_t packed_blocked_bytes(int rows, int cols) {
  const int64_t mt = (rows + BM - 1) / BM, kbt = (cols + BK - 1) / BK;
  return (size_t)(mt * kbt * BM * BK * 2);
}

cudaError_t pack_blocked(const __nv_bfloat16* w, int rows, int cols, int64_t ld, __nv_bfloat16* out, cudaStream_t s) {
  const int kbt = (cols + BK - 1) / BK;
  const int64_t n_vec = (int64_t)packed_blocked_bytes(rows, cols) / 16;
  pack_blocked_kernel<<<(unsigned)((n_vec + 255) / 256 < 4096 ? (n_vec + 255) / 256 : 4096), 256, 0, s>>>(
      w, rows, cols, ld, out, kbt, n_vec);
  return cudaGetLastError();
}

#define SSM_GEMM_KERNELS (const void*)gemm_tc_kernel<0>, (const void*)gemm_tc_kernel<1>, (const void*)gemm_tc_kernel<1, 3>, \
    (const void*)gemm_tc_kernel<1, 4>, (const void*)gemm_tc_kernel<2>, (const void*)gemm_tc_kernel<6>, \
    (const void*)gemm_tc_kernel<7>, (const void*)gemm_tc_kernel<0, XP_NT, 2>, (const void*)gemm_tc_kernel<6, XP_NT, 2>, \
    (const void*)gemm_tc_kernel<7, XP_NT, 2>

// CTA pairs that can be co-resident (one 227 KB CTA per SM): 2-CTA clusters are placed inside a GPC,
// so this can be below num_sms / 2.  Queried once.
int max_pairs() {
  static int pairs = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaFuncSetAttribute((const void*)gemm_tc_kernel<0, XP_NT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) == cudaSuccess &&
        cudaOccupancyMaxActiveClusters(&n, (const void*)gemm_tc_kernel<0, XP_NT, 2>, &cfg) == cudaSuccess)
      pairs = n;
    else
      pairs = 0;
    cudaGetLastError();
  });
  return pairs;
}

cudaError_t preload_gemm_tc() {
  cudaError_t e = cudaSuccess;
  cudaFuncAttributes a;
  for (const void* f : {SSM_GEMM_KERNELS}) {
    if ((e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES)) != cudaSuccess) return e;
    if ((e = cudaFuncGetAttributes(&a, f)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

bool gemm_tc_supported(const void* A, int64_t lda, const void* B, int64_t ldb) {
  return ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0) &&
         ((lda * 2) % 16 == 0) && ((ldb * 2) % 16 == 0) && get_encode() != nullptr;
}

cudaError_t gemm_tc_bf16(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb, int M, int N,
                         int K, int ksplit, const Epilogue& epi, int num_sms, cudaStream_t s, bool a_indep,
                         const __nv_bfloat16* A_blocked) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  // CTA pair (cta_group::2, M = 256 tiles) for the large non-transposed prefill GEMMs: in_proj,
  // out_proj (fp32 residual add or int8 quantisation) and the generic stores; t_gemm_pair forces
  // it on (1) or off (0) for tests and A/B runs
  const bool pair_ok = !epi.trans && ksplit <= 1 && !A_blocked && !a_indep && M > BM && N > 32 &&
                       (epi.kind == EPI_STORE_BF16 || epi.kind == EPI_STORE_F32 || epi.kind == EPI_ADD_F32 ||
                        epi.kind == EPI_QUANT_I8 || epi.kind == EPI_SOFTPLUS_BF16 || epi.kind == EPI_SPLIT_DBC);
  // (measured, Mamba-2.8B prefill chunk of 32768 tokens: in_proj 1356 -> 1209 us, out_proj 690 -> 643 us,
  // x_proj 86 -> 82 us; the K = 160 dt_proj 139 -> 164 us stays on single CTAs)
  const bool pair_default = M >= 4096 && K >= 1024 && N >= 128 && epi.kind != EPI_SOFTPLUS_BF16;
  const int CG = (pair_ok && (t_gemm_pair > 0 || (t_gemm_pair < 0 && pair_default)) && max_pairs() > 0) ? 2 : 1;
  // BN: multiple of 32 in [32, 256] (UMMA needs N % 16 == 0; the epilogue drains TMEM in
  // 32-column chunks) covering N in as few tiles as possible; N <= 16: one 16-column UMMA tile
  // (decode batches) halves the B operand and its smem
  int n_tiles = (N + BN_MAX - 1) / BN_MAX;
  int BN = (N + n_tiles - 1) / n_tiles;
  BN = BN <= 16 ? 16 : (BN + 31) / 32 * 32;
  if (epi.kind == EPI_QUANT_I8 && epi.qblk > 0) BN = (BN + epi.qblk - 1) / epi.qblk * epi.qblk;  // whole blocks
  n_tiles = (N + BN - 1) / BN;
  TileSched ts;
  ts.grp = CG;
  ts.m_tiles = (M + BM * CG - 1) / (BM * CG);
  ts.n_tiles = n_tiles;
  ts.kb_total = (K + BK - 1) / BK;
  if (ksplit < 1) ksplit = 1;
  if (ksplit > ts.kb_total) ksplit = ts.kb_total;
  ts.kbs = (ts.kb_total + ksplit - 1) / ksplit;
  ts.ksplit = (ts.kb_total + ts.kbs - 1) / ts.kbs;
  ts.units = ts.m_tiles * ts.n_tiles * ts.ksplit;
  if (ts.ksplit > 1 && epi.kind != EPI_ATOMIC_F32) return cudaErrorInvalidValue;

  CUtensorMap ma, mb;
  if (!make_map(&mb, B, N, K, ldb, BN / CG)) return cudaErrorInvalidValue;
  if (A_blocked) {
    if ((reinterpret_cast<uintptr_t>(A_blocked) & 127) != 0) return cudaErrorInvalidValue;
    ma = mb;  // unused: A is fetched by 1D bulk copies
  } else if (!make_map(&ma, A, M, K, lda, BM)) {
    return cudaErrorInvalidValue;
  }
  static bool attr_set = false;
  if (!attr_set) {
    for (const void* f : {SSM_GEMM_KERNELS}) {
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  // k-blocks per stage: skinny-N (weight-streaming) GEMMs fetch longer contiguous row segments
  // (decode, N = batch <= 32: 4 k-blocks = 64 KB of weights per stage; measured 39.4 -> 38.1 us per
  // Mamba-2.8B decode layer vs 2, fewer ring turnarounds per CTA)
  int kbs = BN <= 32 ? 4 : BN <= 64 ? 2 : 1;
  CtaRes cr;
  cr.ring = RING_BYTES;
  cr.acc_stride = BN_MAX;
  cr.tmem_cols = 512;
  cr.a_indep = a_indep ? 1 : 0;
  // Skinny-N (decode, weight-streaming) GEMMs take a smaller footprint: a 160 KB ring and a TMEM
  // allocation of 2 x BN columns, so the neighbouring kernels' CTAs (PDL: launched early, their
  // weight / state loads issued before griddepcontrol.wait) can be co-resident on the SM.
  // Measured 40.4 -> 37.7 us per Mamba-2.8B decode layer (stream rate unchanged); 144 and 176 KB
  // rings measured slower (39.2 / 38.8 us).
  if (BN <= 32) {
    cr.ring = 160 * 1024;
    int cols = 32;
    while (cols < 2 * BN) cols *= 2;
    cr.tmem_cols = cols;
    cr.acc_stride = cols / 2;
  }
  int extra = 0;
  if (epi.kind == EPI_DECODE_INPROJ) {
    // fused decode in_proj: one 32-column accumulator per tile, N <= 32 tokens, P <= 320 (even),
    // tiles inside one head, window of <= 3 cached taps
    if (!epi.trans || N > 32 || BN > 32 || epi.P > 8 * 8 * XP_NT || (epi.P & 1) || epi.K < 2 || epi.K > 4 ||
        epi.cph % BM || M != 2 * epi.Ek || ts.ksplit != 1)
      return cudaErrorInvalidValue;
    extra = SU_BYTES + 128;  // u tile
    cr.ring -= SU_BYTES + 128;
  }
  if (epi.kind == EPI_QUANT_I8) {
    // whole qblk blocks inside every tile, 16-B aligned code rows, <= 8 chunks of amax per row
    if (epi.trans || ts.ksplit != 1 || !epi.qs || BN > 256 || BN % 32 || N % epi.qblk ||
        !(epi.qblk == 32 || epi.qblk == 64 || epi.qblk == 128 || epi.qblk == 256) || BN % epi.qblk ||
        epi.ldc % 16 || (reinterpret_cast<uintptr_t>(epi.C) & 15))
      return cudaErrorInvalidValue;
    extra = 128 * 8 * 4;  // s_am
    cr.ring -= extra;
  }
  if (!epi.trans && epi.kind == EPI_SOFTPLUS_BF16) {  // VAR 6: bias + per-warp row staging in shared memory
    if (N % 8 || (epi.ldc * 2) % 16 || (reinterpret_cast<uintptr_t>(epi.C) & 15)) return cudaErrorInvalidValue;
    extra = (N * 4 + 127) / 128 * 128 + 8 * 32 * 144;
    cr.ring -= extra;
  }
  if (epi.kind == EPI_SPLIT_DBC &&
      (epi.trans || ts.ksplit != 1 || epi.dbc_R % 32 || epi.dbc_P % 32 || epi.dbc_R >= epi.dbc_P || N % epi.dbc_P ||
       epi.dbc_M != M || (reinterpret_cast<uintptr_t>(epi.dbc_low) & 15) || (reinterpret_cast<uintptr_t>(epi.dbc_bc) & 15)))
    return cudaErrorInvalidValue;
  if (epi.zero && (reinterpret_cast<uintptr_t>(epi.zero) & 15)) return cudaErrorInvalidValue;
  while (kbs > 1 && num_stages(BN / CG, kbs, cr.ring) < 2) --kbs;
  const int smem_bytes = 1024 + cr.ring + 512 + extra;
  int grid = ts.units < num_sms ? ts.units : num_sms;
  if (CG == 2) {
    const int mp = std::min(num_sms / 2, max_pairs());
    grid = 2 * (ts.units < mp ? ts.units : mp);
  }
  // kernel variant (see gemm_tc_kernel): the decode GEMMs and the prefill dt_proj on their own
  // instantiations (fixed-kind in_proj / out_proj variants measured 2-3% slower than the all-paths
  // kernel, x_proj equal; the dt_proj one 249 -> 230 us)
  int var = 0;
  if (epi.kind == EPI_DECODE_INPROJ) var = 1;
  else if (epi.kind == EPI_ATOMIC_F32 && epi.trans && BN <= 32) var = 2;
  else if (!epi.trans && epi.kind == EPI_SOFTPLUS_BF16) var = 6;
  else if (epi.kind == EPI_QUANT_I8) var = 7;
  if (epi.rss && (var == 1 || var == 6)) return cudaErrorInvalidValue;  // no row scale in those epilogues
  if (epi.cpy && (epi.kind != EPI_ADD_F32 || epi.trans || !epi.ssq || ts.ksplit > 1)) return cudaErrorInvalidValue;
  auto kfn = var == 2 ? gemm_tc_kernel<2> : var == 6 ? gemm_tc_kernel<6> : var == 7 ? gemm_tc_kernel<7> : gemm_tc_kernel<0>;
  if (var == 1) kfn = epi.P <= 64 * 3 ? gemm_tc_kernel<1, 3> : epi.P <= 64 * 4 ? gemm_tc_kernel<1, 4> : gemm_tc_kernel<1>;
  cudaError_t e_;
  if (CG == 2) {
    kfn = var == 6 ? gemm_tc_kernel<6, XP_NT, 2> : var == 7 ? gemm_tc_kernel<7, XP_NT, 2> : gemm_tc_kernel<0, XP_NT, 2>;
    e_ = launch_cluster(kfn, grid, var_threads(var), smem_bytes, s, 2, ma, mb, M, N, BN, kbs, ts, epi, A_blocked, lda, K,
                        cr, 0);
  } else {
    e_ = launch(kfn, grid, var_threads(var), smem_bytes, s, ma, mb, M, N, BN, kbs, ts, epi, A_blocked, lda, K, cr,
                A_blocked ? 1 : 0);
  }
  if (e_ != cudaSuccess) return e_;
  return cudaGetLastError();
}

}  // namespace ssm
