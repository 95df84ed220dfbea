// ssd.cu — the Mamba-2 (SSD) mixer's rank-local kernels (PAPER.md:116,
// 367: "the same high-level mixer pipeline (projection, convolution, state update, gating, output
// projection)").  The projections run on the tcgen05 GEMM and the causal conv on the Mamba-1
// conv kernels (kernels.cu) over the x|B|C channels; this file holds
//   m2_scan         the scalar-A-per-head selective scan: h[p, n] <- exp(dt A) h + dt x[p] B[n],
//                   y[p] = C.h + D x[p]; one CTA per (head, sequence), 256 threads = 64 head
//                   channels x 4 contiguous quarters of the 128 states (32 fp32 states in
//                   registers per thread), token tiles of x, B, C, dt staged by cp.async;
//                   m2_scan_step: the L = 1 decode step as a coalesced stream over the state rows
//   m2_gate_ss      g = y SiLU(z) (fp32, in place) and the row's sum of squares (all-reduced
//                   over the ranks by the caller at TP > 1: the gated RMSNorm spans d_inner)
//   m2_norm_apply   o = g / sqrt(ss / E + eps) * w (bf16), the out_proj's input
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace ssm {
namespace {

constexpr int M2_P = 64, M2_Q = 4, M2_THREADS = M2_P * M2_Q, M2_TT = 16, M2_NMAX = 128;

// proj [M][ldp] bf16: dt raw at column dt_col + h; u [M][ldu] bf16: x at x_col + h P, B at b_col,
// C at c_col (group g of the head: + g N).  h_state [batch][Hk][P][N] fp32 in place; y [M][Ek] fp32.
template <int N>
__global__ void __launch_bounds__(M2_THREADS) m2_scan_kernel(
    const __nv_bfloat16* __restrict__ proj, int64_t ldp, int dt_col, const __nv_bfloat16* __restrict__ u,
    int64_t ldu, int b_col, int c_col, int heads_per_group, const float* __restrict__ dt_bias,
    const float* __restrict__ a_log, const float* __restrict__ d_skip, float* __restrict__ hstate,
    float* __restrict__ y, int64_t ldy, int L, int Hk) {
  constexpr int NPT = N / M2_Q;  // states per thread
  __shared__ __align__(16) __nv_bfloat16 sx[2][M2_TT][M2_P];
  __shared__ __align__(16) __nv_bfloat16 sb[2][M2_TT][N];
  __shared__ __align__(16) __nv_bfloat16 sc[2][M2_TT][N];
  __shared__ float sdt[2][M2_TT];
  pdl_trigger();
  const int h = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, p = tid >> 2, q = tid & 3;
  const int g = h / heads_per_group;
  const int64_t row0 = (int64_t)b * L;
  // the head's weights first (never written by a kernel), then wait for the predecessor's outputs
  const float A = -expf(a_log[h]) * 1.4426950408889634f;  // log2e-scaled: exp(dt A) = 2^(dt A')
  const float bias = dt_bias[h], Dh = d_skip[h];
  pdl_wait();
  float hs[NPT];
  // thread q owns the contiguous states [NPT q, NPT q + NPT): the 4 quarter-threads of a channel read
  // its 512-B state row as one coalesced run of float4s (an interleaved n = q + 4 j ownership made the
  // decode step's state read + write 0.22 of HBM)
  float* hp = hstate + (((int64_t)b * Hk + h) * M2_P + p) * N + NPT * q;
#pragma unroll
  for (int j = 0; j < NPT; j += 4) {
    const float4 v = *reinterpret_cast<const float4*>(hp + j);
    hs[j] = v.x; hs[j + 1] = v.y; hs[j + 2] = v.z; hs[j + 3] = v.w;
  }
  auto load_tile = [&](int buf, int t0) {
    // x: 16 rows x 64 bf16 (8 chunks of 16 B); B, C: 16 rows x N bf16 (N / 8 chunks); dt: 16 values
    constexpr int XC = M2_P / 8, BCC = N / 8;
    for (int i = tid; i < M2_TT * (XC + 2 * BCC); i += M2_THREADS) {
      const int r = i / (XC + 2 * BCC), c = i % (XC + 2 * BCC);
      const int t = t0 + r;
      const bool ok = t < L;
      const int64_t row = row0 + (ok ? t : 0);
      if (c < XC) cp_async16(&sx[buf][r][c * 8], u + row * ldu + (int64_t)h * M2_P + c * 8, ok);
      else if (c < XC + BCC) cp_async16(&sb[buf][r][(c - XC) * 8], u + row * ldu + b_col + (int64_t)g * N + (c - XC) * 8, ok);
      else cp_async16(&sc[buf][r][(c - XC - BCC) * 8], u + row * ldu + c_col + (int64_t)g * N + (c - XC - BCC) * 8, ok);
    }
    if (tid < M2_TT) {
      const int t = t0 + tid;
      float v = 0.f;
      if (t < L) {
        const float raw = __bfloat162float(proj[(row0 + t) * ldp + dt_col + h]) + bias;
        v = softplus(raw);
      }
      sdt[buf][tid] = v;
    }
  };
  const int ntiles = (L + M2_TT - 1) / M2_TT;
  load_tile(0, 0);
  cp_async_commit();
  for (int it = 0; it < ntiles; ++it) {
    const int buf = it & 1;
    if (it + 1 < ntiles) {
      load_tile(buf ^ 1, (it + 1) * M2_TT);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int t0 = it * M2_TT, tn = min(M2_TT, L - t0);
    for (int r = 0; r < tn; ++r) {
      const float dt = sdt[buf][r];
      const float dA = ex2_approx(dt * A);
      const float xv = __bfloat162float(sx[buf][r][p]);
      const float dtx = dt * xv;
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int n = NPT * q + j;
        hs[j] = fmaf(dA, hs[j], dtx * __bfloat162float(sb[buf][r][n]));
        acc = fmaf(__bfloat162float(sc[buf][r][n]), hs[j], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (q == 0) y[(row0 + t0 + r) * ldy + (int64_t)h * M2_P + p] = fmaf(Dh, xv, acc);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NPT; j += 4) *reinterpret_cast<float4*>(hp + j) = make_float4(hs[j], hs[j + 1], hs[j + 2], hs[j + 3]);
}

// The decode step (L = 1): the state read + write (B Hk P N fp32 each way; 42 MB per Mamba-2-2.7B
// layer at batch 16) is the whole cost, so the work is spread as a stream rather than one CTA per
// (head, sequence) (that form, 66 registers x 256 threads, fits 3 CTAs per SM and runs 1280 CTAs in
// ~3 latency-bound waves): N / 8 lanes per state row (b, h, p), 8 states per lane (two float4 of h,
// one 16-B run each of B and C), the row's C.h by shuffles inside the lane group.
template <int N>
__global__ void __launch_bounds__(256) m2_scan_step_kernel(
    const __nv_bfloat16* __restrict__ proj, int64_t ldp, int dt_col, const __nv_bfloat16* __restrict__ u,
    int64_t ldu, int b_col, int c_col, int heads_per_group, const float* __restrict__ dt_bias,
    const float* __restrict__ a_log, const float* __restrict__ d_skip, float* __restrict__ hstate,
    float* __restrict__ y, int64_t ldy, int64_t rows, int Hk) {
  constexpr int LPR = N / 8;  // lanes per state row (a power of two dividing 32)
  pdl_trigger();
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR;  // (b, h, p)
  const int sub = threadIdx.x % LPR;
  const bool live = row < rows;
  const int64_t rr = live ? row : 0;
  const int p = (int)(rr % M2_P);
  const int h = (int)((rr / M2_P) % Hk);
  const int64_t b = rr / ((int64_t)M2_P * Hk);
  const int g = h / heads_per_group;
  const float A = -expf(a_log[h]) * 1.4426950408889634f;
  const float bias = dt_bias[h], Dh = d_skip[h];
  pdl_wait();
  float* hp = hstate + rr * N + 8 * sub;
  const float4 h0 = *reinterpret_cast<const float4*>(hp), h1 = *reinterpret_cast<const float4*>(hp + 4);
  const uint4 bv = *reinterpret_cast<const uint4*>(u + b * ldu + b_col + (int64_t)g * N + 8 * sub);
  const uint4 cv = *reinterpret_cast<const uint4*>(u + b * ldu + c_col + (int64_t)g * N + 8 * sub);
  const float xv = __bfloat162float(u[b * ldu + (int64_t)h * M2_P + p]);
  const float dt = softplus(__bfloat162float(proj[b * ldp + dt_col + h]) + bias);
  const float dA = ex2_approx(dt * A), dtx = dt * xv;
  float hs[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
  const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&bv);
  const __nv_bfloat16* cc = reinterpret_cast<const __nv_bfloat16*>(&cv);
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    hs[j] = fmaf(dA, hs[j], dtx * __bfloat162float(bb[j]));
    acc = fmaf(__bfloat162float(cc[j]), hs[j], acc);
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (!live) return;
  *reinterpret_cast<float4*>(hp) = make_float4(hs[0], hs[1], hs[2], hs[3]);
  *reinterpret_cast<float4*>(hp + 4) = make_float4(hs[4], hs[5], hs[6], hs[7]);
  if (sub == 0) y[b * ldy + (int64_t)h * M2_P + p] = fmaf(Dh, xv, acc);
}

// g = y * SiLU(z) in place (y fp32 [M][Ek], z bf16 at proj[m][z_col..]); ss[m] = sum g^2
__global__ void __launch_bounds__(256) m2_gate_ss_kernel(float* __restrict__ y, int Ek,
                                                         const __nv_bfloat16* __restrict__ proj, int64_t ldp,
                                                         float* __restrict__ ss) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8];
  const int64_t m = blockIdx.x;
  float s = 0.f;
  for (int c = threadIdx.x; c < Ek; c += 256) {
    const float z = __bfloat162float(proj[m * ldp + c]);
    const float gv = y[m * Ek + c] * (z / (1.0f + expf(-z)));
    y[m * Ek + c] = gv;
    s = fmaf(gv, gv, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < 8; ++i) t += red[i];
    ss[m] = t;
  }
}

// o = g / sqrt(ss / E + eps) * w -> bf16
__global__ void m2_norm_apply_kernel(const float* __restrict__ g, int Ek, const float* __restrict__ ss, int E,
                                     float eps, const float* __restrict__ w, __nv_bfloat16* __restrict__ o, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / Ek;
    const int c = (int)(i % Ek);
    o[i] = __float2bfloat16_rn(g[i] * (1.0f / sqrtf(ss[m] / (float)E + eps)) * w[c]);
  }
}

}  // namespace

cudaError_t launch_m2_scan(const __nv_bfloat16* proj, int64_t ldp, int dt_col, const __nv_bfloat16* u, int64_t ldu,
                           int b_col, int c_col, int heads_per_group, const float* dt_bias, const float* a_log,
                           const float* d_skip, float* hstate, float* y, int64_t ldy, int batch, int L, int Hk, int P,
                           int N, cudaStream_t s) {
  if (batch <= 0 || L <= 0) return cudaSuccess;
  if (P != M2_P) return cudaErrorInvalidValue;
  cudaError_t e;
  if (L == 1) {
    const int64_t rows = (int64_t)batch * Hk * M2_P;
    const unsigned blocks = (unsigned)((rows * (N / 8) + 255) / 256);
    switch (N) {
      case 128: e = launch(m2_scan_step_kernel<128>, blocks, 256, 0, s, proj, ldp, dt_col, u, ldu, b_col, c_col,
                           heads_per_group, dt_bias, a_log, d_skip, hstate, y, ldy, rows, Hk); break;
      case 64: e = launch(m2_scan_step_kernel<64>, blocks, 256, 0, s, proj, ldp, dt_col, u, ldu, b_col, c_col,
                          heads_per_group, dt_bias, a_log, d_skip, hstate, y, ldy, rows, Hk); break;
      case 16: e = launch(m2_scan_step_kernel<16>, blocks, 256, 0, s, proj, ldp, dt_col, u, ldu, b_col, c_col,
                          heads_per_group, dt_bias, a_log, d_skip, hstate, y, ldy, rows, Hk); break;
      default: return cudaErrorInvalidValue;
    }
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  dim3 grid(Hk, batch);
  switch (N) {
    case 128: e = launch(m2_scan_kernel<128>, grid, M2_THREADS, 0, s, proj, ldp, dt_col, u, ldu, b_col, c_col,
                         heads_per_group, dt_bias, a_log, d_skip, hstate, y, ldy, L, Hk); break;
    case 64: e = launch(m2_scan_kernel<64>, grid, M2_THREADS, 0, s, proj, ldp, dt_col, u, ldu, b_col, c_col,
                        heads_per_group, dt_bias, a_log, d_skip, hstate, y, ldy, L, Hk); break;
    case 16: e = launch(m2_scan_kernel<16>, grid, M2_THREADS, 0, s, proj, ldp, dt_col, u, ldu, b_col, c_col,
                        heads_per_group, dt_bias, a_log, d_skip, hstate, y, ldy, L, Hk); break;
    default: return cudaErrorInvalidValue;
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_m2_gate_ss(float* y, int Ek, const __nv_bfloat16* proj, int64_t ldp, float* ss, int64_t M,
                              cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  cudaError_t e = launch(m2_gate_ss_kernel, (unsigned)M, 256, 0, s, y, Ek, proj, ldp, ss);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_m2_norm_apply(const float* g, int Ek, const float* ss, int E, float eps, const float* w,
                                 __nv_bfloat16* o, int64_t M, cudaStream_t s) {
  const int64_t n = M * Ek;
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  cudaError_t e = launch(m2_norm_apply_kernel, (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s, g, Ek,
                         ss, E, eps, w, o, n);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t preload_ssd() {
  cudaFuncAttributes a;
  for (const void* f : {(const void*)m2_scan_kernel<128>, (const void*)m2_scan_kernel<64>,
                        (const void*)m2_scan_kernel<16>, (const void*)m2_scan_step_kernel<128>,
                        (const void*)m2_scan_step_kernel<64>, (const void*)m2_scan_step_kernel<16>,
                        (const void*)m2_gate_ss_kernel,
                        (const void*)m2_norm_apply_kernel}) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ssm
