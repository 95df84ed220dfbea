// attn.cu — kernels of Zamba's shared transformer block:
//   rmsnorm_cat   x = RMSNorm(concat(h, h0)) * w (bf16 out), and RMSNorm(h + t) for the hybrid
//                 layer's Mamba input
//   kv_append     K, V rows of this call -> the KV cache at the device-side length
//   attn          causal softmax attention over the cache, flash-style (online softmax), bf16
//                 operands on mma.sync m16n8k16 with fp32 accumulation; 64 query rows per CTA,
//                 8 warps = 4 row groups x 2 halves of the head dimension (O stays in registers)
//   gelu_mul      m = GELU(gate) * up (erf GELU), bf16
//   cast          fp32 -> bf16
// The projections (qkv, o, gate/up, down, linear) run on the tcgen05 GEMM (gemm_tcgen05.cu).
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace ssm {
namespace {

// ---------------------------------------------------------------- RMSNorm of a concatenation / sum
// One 256-thread block per row.  mode 0: row = concat(a[m], b[m]) of width 2D; mode 1: row =
// a[m] + b[m] of width D (b may be NULL).  y = row / sqrt(mean(row^2) + eps) * w (w may be NULL).
constexpr int RN_THREADS = 256, RN_MAXV = 8;  // <= 8192 floats per row
__global__ void __launch_bounds__(RN_THREADS) rmsnorm2_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                              int mode, const float* __restrict__ w, float eps,
                                                              __nv_bfloat16* __restrict__ y, int D) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[RN_THREADS / 32];
  const int64_t row = blockIdx.x;
  const int W = mode == 0 ? 2 * D : D;
  const int nv = W / 4, dv = D / 4;
  float4 v[RN_MAXV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < RN_MAXV; ++i) {
    const int k = threadIdx.x + i * RN_THREADS;
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < nv) {
      if (mode == 0) {
        v[i] = k < dv ? reinterpret_cast<const float4*>(a + row * D)[k] : reinterpret_cast<const float4*>(b + row * D)[k - dv];
      } else {
        v[i] = reinterpret_cast<const float4*>(a + row * D)[k];
        if (b) {
          const float4 t = reinterpret_cast<const float4*>(b + row * D)[k];
          v[i].x += t.x; v[i].y += t.y; v[i].z += t.z; v[i].w += t.w;
        }
      }
      ss = fmaf(v[i].x, v[i].x, ss); ss = fmaf(v[i].y, v[i].y, ss);
      ss = fmaf(v[i].z, v[i].z, ss); ss = fmaf(v[i].w, v[i].w, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < RN_THREADS / 32; ++i) tot += red[i];
  const float rs = 1.0f / sqrtf(tot / (float)W + eps);
#pragma unroll
  for (int i = 0; i < RN_MAXV; ++i) {
    const int k = threadIdx.x + i * RN_THREADS;
    if (k < nv) {
      float4 ww = make_float4(1.f, 1.f, 1.f, 1.f);
      if (w) ww = reinterpret_cast<const float4*>(w)[k];
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * rs * ww.x, v[i].y * rs * ww.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * rs * ww.z, v[i].w * rs * ww.w);
      uint2 pk;
      pk.x = *reinterpret_cast<const uint32_t*>(&lo);
      pk.y = *reinterpret_cast<const uint32_t*>(&hi);
      reinterpret_cast<uint2*>(y + row * W)[k] = pk;
    }
  }
}

// ---------------------------------------------------------------- KV cache append
// qkv [B*L][3 Hk d] (q | k | v); cache K, V [B][Tmax][Hk][d]; rows land at t = len + l.
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ qkv, const int* __restrict__ len, int L, int Hk,
                                 int d, int Tmax, __nv_bfloat16* __restrict__ Kc, __nv_bfloat16* __restrict__ Vc,
                                 int64_t nvec, int* __restrict__ err) {
  pdl_trigger();
  pdl_wait();
  const int t0 = *reinterpret_cast<const volatile int*>(len);   // (volatile: not hoisted above the PDL wait)
  if (t0 + L > Tmax) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *err = 1;
    return;
  }
  const int dv = d / 8;  // 16-B vectors per head row
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % dv);
    const int64_t r = i / dv;           // (row m, head h)
    const int h = (int)(r % Hk);
    const int64_t m = r / Hk;
    const int64_t b = m / L, l = m % L;
    const uint4* src = reinterpret_cast<const uint4*>(qkv + m * 3 * Hk * d);
    const int64_t dst = (((b * Tmax) + t0 + l) * Hk + h) * dv + j;
    reinterpret_cast<uint4*>(Kc)[dst] = src[(int64_t)(Hk + h) * dv + j];
    reinterpret_cast<uint4*>(Vc)[dst] = src[(int64_t)(2 * Hk + h) * dv + j];
  }
}

__global__ void kv_advance_kernel(int* len, int L, int Tmax) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    volatile int* v = reinterpret_cast<volatile int*>(len);
    const int n = *v + L;
    *v = n < Tmax ? n : Tmax;  // saturating (an overflowing append wrote nothing and set the error word)
  }
}

// ---------------------------------------------------------------- causal flash attention
// q rows at positions t0 + l (l < L) of batch b attend to cache rows 0 .. t0 + l.  d = head dim
// (multiple of 16, <= 464); DH = O columns per warp = d / 2 (multiple of 8).
constexpr int AQ = 64, AK = 64, AT = 256;  // query rows, keys per tile, threads
template <int D_>
struct AttnSmem {
  static constexpr int PITCH = D_ + 8;  // bf16 elements: 16-B rows, conflict-free ldmatrix
  static constexpr int BYTES = 3 * AQ * PITCH * 2;
};

template <int D_>
__global__ void __launch_bounds__(AT, 1) attn_kernel(const __nv_bfloat16* __restrict__ qkv, const int* __restrict__ len,
                                                     const __nv_bfloat16* __restrict__ Kc,
                                                     const __nv_bfloat16* __restrict__ Vc, int L, int Hk, int Tmax,
                                                     float scale_log2, __nv_bfloat16* __restrict__ out) {
  constexpr int P = AttnSmem<D_>::PITCH;
  constexpr int DH = D_ / 2, NT = DH / 8, KS = D_ / 16, CV = D_ / 8;  // O n-tiles per warp, k-steps, 16-B chunks
  extern __shared__ __align__(16) uint8_t asm_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(asm_raw);
  __nv_bfloat16* sK = sQ + AQ * P;
  __nv_bfloat16* sV = sK + AK * P;
  pdl_trigger();
  pdl_wait();
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qg = warp & 3, dh = warp >> 2;
  // the cache already holds this call's rows; a volatile read, so the compiler cannot hoist it as a
  // read-only (LDG.CONSTANT) load above griddepcontrol.wait -- the length is written by the
  // predecessor kernel
  const int t0 = *reinterpret_cast<const volatile int*>(len) - L;
  const int T = t0 + L;
  const int q_lo = qt * AQ;
  const int q_hi = min(L, q_lo + AQ);
  const int64_t ldq = 3 * (int64_t)Hk * D_;
  // Q tile
  for (int i = tid; i < AQ * CV; i += AT) {
    const int r = i / CV, c = i % CV;
    const int l = q_lo + r;
    cp_async16(sQ + r * P + c * 8, qkv + ((int64_t)b * L + (l < L ? l : 0)) * ldq + (int64_t)h * D_ + c * 8, l < L);
  }
  auto load_kv = [&](__nv_bfloat16* dst, const __nv_bfloat16* cache, int k0) {
    for (int i = tid; i < AK * CV; i += AT) {
      const int r = i / CV, c = i % CV;
      const int t = k0 + r;
      cp_async16(dst + r * P + c * 8, cache + (((int64_t)b * Tmax + (t < T ? t : 0)) * Hk + h) * D_ + c * 8, t < T);
    }
  };
  const int kend = min(T, t0 + q_hi);      // keys needed by the last query row of the tile
  const int nkt = (kend + AK - 1) / AK;
  load_kv(sK, Kc, 0);
  cp_async_commit();                       // group: Q + K0
  load_kv(sV, Vc, 0);
  cp_async_commit();                       // group: V0
  float o[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int r0 = qg * 16 + (lane >> 2);    // this lane's rows r0, r0 + 8 of the tile
  const int qp0 = t0 + q_lo + r0, qp1 = qp0 + 8;
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<1>();
    __syncthreads();                       // K[kt] (and Q) visible
    // ---- S = Q K^T for 16 rows x 64 keys
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll 1
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t a[4];
      ldmatrix_x4(a, sQ + (qg * 16 + (lane & 15)) * P + ks * 16 + (lane >> 4) * 8);
#pragma unroll
      for (int n = 0; n < 8; n += 2) {
        uint32_t bb[4];  // keys 8n .. 8n+15: (k lo, k hi) of n-tile n, then of n-tile n + 1
        ldmatrix_x4(bb, sK + (n * 8 + (lane & 7) + ((lane >> 4) << 3)) * P + ks * 16 + ((lane >> 3) & 1) * 8);
        mma_16816_bf16(s[n], a, bb[0], bb[1]);
        mma_16816_bf16(s[n + 1], a, bb[2], bb[3]);
      }
    }
    __syncthreads();                       // every warp is done with K[kt]
    if (kt + 1 < nkt) load_kv(sK, Kc, (kt + 1) * AK);
    cp_async_commit();
    // ---- causal mask, online softmax (base 2)
    const int k0 = kt * AK;
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + n * 8 + 2 * (lane & 3) + (e & 1);
        const int qp = (e < 2) ? qp0 : qp1;
        const float v = (key <= qp && key < T) ? s[n][e] * scale_log2 : -INFINITY;
        s[n][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
    }
    float alpha[2], ps[2] = {0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 2; ++i) alpha[i] = mx[i] == -INFINITY ? 1.f : ex2_approx(mrow[i] - mx[i]);
    uint32_t pa[4][4];  // P as A fragments, 4 k-steps of 16 keys
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m = mx[e >> 1];
        p[e] = m == -INFINITY ? 0.f : ex2_approx(s[n][e] - m);
        ps[e >> 1] += p[e];
      }
      const __nv_bfloat162 lo = __floats2bfloat162_rn(p[0], p[1]), hi = __floats2bfloat162_rn(p[2], p[3]);
      pa[n >> 1][(n & 1) * 2 + 0] = *reinterpret_cast<const uint32_t*>(&lo);
      pa[n >> 1][(n & 1) * 2 + 1] = *reinterpret_cast<const uint32_t*>(&hi);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      ps[i] += __shfl_xor_sync(0xffffffffu, ps[i], 1);
      ps[i] += __shfl_xor_sync(0xffffffffu, ps[i], 2);
      lrow[i] = lrow[i] * alpha[i] + ps[i];
      mrow[i] = mx[i];
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      o[i][0] *= alpha[0]; o[i][1] *= alpha[0];
      o[i][2] *= alpha[1]; o[i][3] *= alpha[1];
    }
    cp_async_wait<1>();
    __syncthreads();                       // V[kt] visible
    // ---- O += P V over this warp's half of the head dimension
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      // A fragment order of m16n8k16: a0 (rows lo, k 0-7), a1 (rows hi, k 0-7), a2 (rows lo, k 8-15), a3 (rows hi, k 8-15)
      const uint32_t a[4] = {pa[ks][0], pa[ks][1], pa[ks][2], pa[ks][3]};
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        uint32_t bb[2];
        ldmatrix_x2_trans(bb, sV + (ks * 16 + (lane & 15)) * P + dh * DH + i * 8);
        mma_16816_bf16(o[i], a, bb[0], bb[1]);
      }
    }
    __syncthreads();                       // every warp is done with V[kt]
    if (kt + 1 < nkt) load_kv(sV, Vc, (kt + 1) * AK);
    cp_async_commit();
  }
  cp_async_wait<0>();
  // ---- normalise and store: rows r0, r0 + 8; columns dh DH + 8 i + 2 (lane % 4)
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int l = q_lo + r0 + 8 * hr;
    if (l >= L) continue;
    const float inv = lrow[hr] > 0.f ? 1.f / lrow[hr] : 0.f;
    __nv_bfloat16* dst = out + ((int64_t)b * L + l) * Hk * D_ + (int64_t)h * D_ + dh * DH + 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const __nv_bfloat162 v = __floats2bfloat162_rn(o[i][2 * hr] * inv, o[i][2 * hr + 1] * inv);
      *reinterpret_cast<__nv_bfloat162*>(dst + i * 8) = v;
    }
  }
}

// ---------------------------------------------------------------- decode attention (L = 1)
// Memory-bound flash decoding: grid (splits, Hk, batch); a 128-thread CTA streams its slice of the
// cache rows of one (b, head); each warp takes keys in groups of 4 (all of their K and V 16-B
// chunks in flight together: a lane owns chunks lane and lane + 32 of a d-wide row), forms the
// scores with a warp reduction and keeps an online softmax and its share of the output; the CTA
// then merges its warps and writes a partial (max, sum, acc[d]) per split, merged by
// attn_dec_combine_kernel.  d % 8 == 0, d <= 512.
constexpr int DEC_THREADS = 128, DEC_G = 4;
__global__ void __launch_bounds__(DEC_THREADS) attn_dec_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                               const int* __restrict__ len,
                                                               const __nv_bfloat16* __restrict__ Kc,
                                                               const __nv_bfloat16* __restrict__ Vc, int Hk, int d,
                                                               int Tmax, float scale_log2, int keys_per_split,
                                                               float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  const int sp = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = *reinterpret_cast<const volatile int*>(len);
  const int nch = d / 8;
  const int k_lo = sp * keys_per_split, k_hi = min(T, k_lo + keys_per_split);
  // q: a lane's two 16-B chunks (lane, lane + 32)
  float q[2][8];
  const __nv_bfloat16* qr = qkv + (int64_t)b * 3 * Hk * d + (int64_t)h * d;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int ch = lane + 32 * c;
    uint4 raw = ch < nch ? reinterpret_cast<const uint4*>(qr)[ch] : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h2[j]);
      q[c][2 * j] = f.x * scale_log2;
      q[c][2 * j + 1] = f.y * scale_log2;
    }
  }
  float m = -INFINITY, l = 0.f, acc[2][8];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[c][j] = 0.f;
  const int64_t row_stride = (int64_t)Hk * d;
  const __nv_bfloat16* Kb = Kc + ((int64_t)b * Tmax) * row_stride + (int64_t)h * d;
  const __nv_bfloat16* Vb = Vc + ((int64_t)b * Tmax) * row_stride + (int64_t)h * d;
  for (int k0 = k_lo + warp * DEC_G; k0 < k_hi; k0 += 4 * DEC_G) {
    uint4 kr[DEC_G][2], vr[DEC_G][2];
#pragma unroll
    for (int g = 0; g < DEC_G; ++g)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int ch = lane + 32 * c;
        const bool ok = k0 + g < k_hi && ch < nch;
        kr[g][c] = ok ? reinterpret_cast<const uint4*>(Kb + (int64_t)(k0 + g) * row_stride)[ch] : make_uint4(0, 0, 0, 0);
        vr[g][c] = ok ? reinterpret_cast<const uint4*>(Vb + (int64_t)(k0 + g) * row_stride)[ch] : make_uint4(0, 0, 0, 0);
      }
    float s[DEC_G];
#pragma unroll
    for (int g = 0; g < DEC_G; ++g) {
      float a = 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kr[g][c]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(k2[j]);
          a = fmaf(q[c][2 * j], f.x, fmaf(q[c][2 * j + 1], f.y, a));
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      s[g] = k0 + g < k_hi ? a : -INFINITY;
    }
    float mn = m;
#pragma unroll
    for (int g = 0; g < DEC_G; ++g) mn = fmaxf(mn, s[g]);
    const float alpha = m == -INFINITY ? 0.f : ex2_approx(m - mn);
    l *= alpha;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[c][j] *= alpha;
#pragma unroll
    for (int g = 0; g < DEC_G; ++g) {
      const float p = s[g] == -INFINITY ? 0.f : ex2_approx(s[g] - mn);
      l += p;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vr[g][c]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(v2[j]);
          acc[c][2 * j] = fmaf(p, f.x, acc[c][2 * j]);
          acc[c][2 * j + 1] = fmaf(p, f.y, acc[c][2 * j + 1]);
        }
      }
    }
    m = mn;
  }
  // merge the 4 warps (shared memory), write the split's partial: [m, l, acc[d]]
  __shared__ float s_m[4], s_l[4];
  __shared__ float s_acc[4][512];
  if (lane == 0) { s_m[warp] = m; s_l[warp] = l; }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int ch = lane + 32 * c;
    if (ch < nch)
#pragma unroll
      for (int j = 0; j < 8; ++j) s_acc[warp][ch * 8 + j] = acc[c][j];
  }
  __syncthreads();
  float M = fmaxf(fmaxf(s_m[0], s_m[1]), fmaxf(s_m[2], s_m[3]));
  float w[4], Lt = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    w[i] = s_m[i] == -INFINITY ? 0.f : ex2_approx(s_m[i] - M);
    Lt += w[i] * s_l[i];
  }
  float* pp = part + (((int64_t)b * Hk + h) * gridDim.x + sp) * (2 + d);
  if (threadIdx.x == 0) { pp[0] = M; pp[1] = Lt; }
  for (int i = threadIdx.x; i < d; i += DEC_THREADS)
    pp[2 + i] = w[0] * s_acc[0][i] + w[1] * s_acc[1][i] + w[2] * s_acc[2][i] + w[3] * s_acc[3][i];
}

__global__ void attn_dec_combine_kernel(const float* __restrict__ part, int splits, int Hk, int d,
                                        __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, b = blockIdx.y;
  const float* pp = part + ((int64_t)b * Hk + h) * splits * (2 + d);
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, pp[s * (2 + d)]);
  float Lt = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float ms = pp[s * (2 + d)];
    Lt += ms == -INFINITY ? 0.f : ex2_approx(ms - M) * pp[s * (2 + d) + 1];
  }
  const float inv = Lt > 0.f ? 1.f / Lt : 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float o = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float ms = pp[s * (2 + d)];
      if (ms != -INFINITY) o = fmaf(ex2_approx(ms - M), pp[s * (2 + d) + 2 + i], o);
    }
    out[((int64_t)b * Hk + h) * d + i] = __float2bfloat16_rn(o * inv);
  }
}

// ---------------------------------------------------------------- MLP gate and cast
// gu [M][2 I] bf16 (gate | up) -> m [M][I] bf16 = GELU(gate) * up, GELU(x) = x Phi(x) (erf form)
__global__ void gelu_mul_kernel(const __nv_bfloat16* __restrict__ gu, int64_t M, int I, __nv_bfloat16* __restrict__ m) {
  pdl_trigger();
  pdl_wait();
  const int iv = I / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * iv; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / iv;
    const int c = (int)(i % iv);
    const uint4 g4 = reinterpret_cast<const uint4*>(gu + r * 2 * I)[c];
    const uint4 u4 = reinterpret_cast<const uint4*>(gu + r * 2 * I + I)[c];
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g4);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u4);
    uint4 o4;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o4);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 g = __bfloat1622float2(g2[j]), u = __bfloat1622float2(u2[j]);
      const float a = 0.5f * g.x * (1.f + erff(g.x * 0.70710678118654752f)) * u.x;
      const float c2 = 0.5f * g.y * (1.f + erff(g.y * 0.70710678118654752f)) * u.y;
      o2[j] = __floats2bfloat162_rn(a, c2);
    }
    reinterpret_cast<uint4*>(m + r * I)[c] = o4;
  }
}

__global__ void cast_bf16_kernel(const float* __restrict__ x, int64_t n4, __nv_bfloat16* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<const uint32_t*>(&lo);
    pk.y = *reinterpret_cast<const uint32_t*>(&hi);
    reinterpret_cast<uint2*>(y)[i] = pk;
  }
}

inline int grid_for(int64_t n, int threads) {
  const int64_t g = (n + threads - 1) / threads;
  return (int)(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

}  // namespace

cudaError_t launch_rmsnorm2(const float* a, const float* b, int mode, const float* w, float eps, __nv_bfloat16* y,
                            int64_t M, int D, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const int W = mode == 0 ? 2 * D : D;
  if (D % 4 || W > RN_THREADS * RN_MAXV * 4) return cudaErrorInvalidValue;
  cudaError_t e = launch(rmsnorm2_kernel, (unsigned)M, RN_THREADS, 0, s, a, b, mode, w, eps, y, D);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_kv_append(const __nv_bfloat16* qkv, const int* len, int batch, int L, int Hk, int d, int Tmax,
                             __nv_bfloat16* K, __nv_bfloat16* V, int* err, cudaStream_t s) {
  if (d % 8) return cudaErrorInvalidValue;
  const int64_t nvec = (int64_t)batch * L * Hk * (d / 8);
  if (nvec <= 0) return cudaSuccess;
  cudaError_t e = launch(kv_append_kernel, grid_for(nvec, 256), 256, 0, s, qkv, len, L, Hk, d, Tmax, K, V, nvec, err);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_kv_advance(int* len, int L, int Tmax, cudaStream_t s) {
  cudaError_t e = launch(kv_advance_kernel, 1, 32, 0, s, len, L, Tmax);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int D_>
static cudaError_t attn_t(const __nv_bfloat16* qkv, const int* len, const __nv_bfloat16* K, const __nv_bfloat16* V,
                          int batch, int L, int Hk, int Tmax, float scale, __nv_bfloat16* out, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_kernel<D_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AttnSmem<D_>::BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((L + AQ - 1) / AQ, Hk, batch);
  cudaError_t e = launch(attn_kernel<D_>, grid, AT, AttnSmem<D_>::BYTES, s, qkv, len, K, V, L, Hk, Tmax,
                         scale * 1.4426950408889634f, out);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_attn(const __nv_bfloat16* qkv, const int* len, const __nv_bfloat16* K, const __nv_bfloat16* V,
                        int batch, int L, int Hk, int d, int Tmax, float scale, __nv_bfloat16* out, cudaStream_t s) {
  if (batch <= 0 || L <= 0) return cudaSuccess;
  switch (d) {
    case 464: return attn_t<464>(qkv, len, K, V, batch, L, Hk, Tmax, scale, out, s);   // Zamba-7B
    case 32: return attn_t<32>(qkv, len, K, V, batch, L, Hk, Tmax, scale, out, s);     // test shapes
    case 64: return attn_t<64>(qkv, len, K, V, batch, L, Hk, Tmax, scale, out, s);
    case 128: return attn_t<128>(qkv, len, K, V, batch, L, Hk, Tmax, scale, out, s);
    default: return cudaErrorInvalidValue;
  }
}

// decode (L = 1): splits chosen so that ~3 CTAs per SM stream the cache; part: workspace of
// batch * Hk * splits * (2 + d) floats (attn_dec_part_floats)
int attn_dec_splits(int batch, int Hk, int Tmax) {
  int sp = (3 * 148 + batch * Hk - 1) / (batch * Hk);
  const int maxsp = (Tmax + 63) / 64;
  if (sp > maxsp) sp = maxsp;
  return sp < 1 ? 1 : sp;
}
size_t attn_dec_part_floats(int batch, int Hk, int d, int Tmax) {
  return (size_t)batch * Hk * attn_dec_splits(batch, Hk, Tmax) * (2 + d);
}
cudaError_t launch_attn_decode(const __nv_bfloat16* qkv, const int* len, const __nv_bfloat16* K, const __nv_bfloat16* V,
                               int batch, int Hk, int d, int Tmax, float scale, float* part, __nv_bfloat16* out,
                               cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  if (d % 8 || d > 512) return cudaErrorInvalidValue;
  const int sp = attn_dec_splits(batch, Hk, Tmax);
  const int kps = (Tmax + sp - 1) / sp;
  cudaError_t e = launch(attn_dec_kernel, dim3(sp, Hk, batch), DEC_THREADS, 0, s, qkv, len, K, V, Hk, d, Tmax,
                         scale * 1.4426950408889634f, kps, part);
  if (e != cudaSuccess) return e;
  e = launch(attn_dec_combine_kernel, dim3(Hk, batch), 128, 0, s, (const float*)part, sp, Hk, d, out);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_gelu_mul(const __nv_bfloat16* gu, int64_t M, int I, __nv_bfloat16* m, cudaStream_t s) {
  if (I % 8) return cudaErrorInvalidValue;
  if (M <= 0) return cudaSuccess;
  cudaError_t e = launch(gelu_mul_kernel, grid_for(M * (I / 8), 256), 256, 0, s, gu, M, I, m);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_cast_bf16(const float* x, int64_t n, __nv_bfloat16* y, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  if (n <= 0) return cudaSuccess;
  cudaError_t e = launch(cast_bf16_kernel, grid_for(n / 4, 256), 256, 0, s, x, n / 4, y);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t preload_attn() {
  cudaFuncAttributes a;
  for (const void* f : {(const void*)rmsnorm2_kernel, (const void*)kv_append_kernel, (const void*)kv_advance_kernel,
                        (const void*)attn_kernel<464>, (const void*)attn_kernel<32>, (const void*)attn_kernel<64>,
                        (const void*)attn_kernel<128>, (const void*)gelu_mul_kernel, (const void*)cast_bf16_kernel,
                        (const void*)attn_dec_kernel, (const void*)attn_dec_combine_kernel}) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ssm
