// kernels.cu — the rank-local mixer kernels of libssmtp (sm_100a) and the
// peer-to-peer all-reduce kernels.  All HBM-bound work: 16-byte vector / cp.async
// loads, token-major activations with channels contiguous.
//
//  conv1d_silu      SURVEY §8(a) a2  causal depthwise conv + SiLU
//  conv_state_upd   a11              conv window of the SSM cache
//  conv_decode      a10              conv update for one token, in place
//  unpack           a4               AR#1 fixed-order sum + dt/B/C split (+Falcon RMSNorm)
//  scan_chunked     a6/a7            selective scan, D skip, SiLU(z) gate, h carried
//  decode_step      a10              dt_proj + softplus + one scan step + gate, h in place
//  quantize/qar     a8/a9            int8 per-block codes, fixed-order dequant-accumulate
//  peer_barrier     a4/a9            epoch flags over NVLink (st.release.sys / ld.acquire.sys)
//  rmsnorm                           pre-norm glue (reading Q16)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "dstep.cuh"

namespace ssm {
namespace {

// ---------------------------------------------------------------- vector IO
template <typename T, int V>
struct Vec;
template <>
struct Vec<__nv_bfloat16, 8> {
  __device__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
    uint4 r = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = r;
  }
};
template <>
struct Vec<float, 4> {
  __device__ static void load(const float* p, float (&v)[4]) {
    float4 r = *reinterpret_cast<const float4*>(p);
    v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
  }
  __device__ static void store(float* p, const float (&v)[4]) { *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]); }
};

template <typename T>
constexpr int vec_of() { return 16 / sizeof(T); }

// ---------------------------------------------------------------- conv1d + SiLU (prefill)
// u[b,t,d] = SiLU(conv_b[d] + sum_j conv_w[d,j] * xt[b, t-K+1+j, d]), xt = conv_state || x.
// One thread per (b, 16-B channel group, CONV_TCH consecutive tokens): conv weights and the
// K-1 window in registers, rows prefetched CONV_PF tokens ahead (software pipelining).  A
// block spans CONV_CG channel groups = a 4-KB contiguous segment of each row (bf16).
constexpr int CONV_CG = 256, CONV_TCH = 16, CONV_PF = 2;
template <typename T, int K, bool FAST>
__global__ void __launch_bounds__(CONV_CG) conv1d_silu_kernel(const T* __restrict__ xz, int64_t ldxz,
                                                              const T* __restrict__ cst, const float* __restrict__ cw,
                                                              const float* __restrict__ cb, T* __restrict__ u,
                                                              int64_t ldu, int L, int Ek) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = vec_of<T>();
  const int cg = blockIdx.x * CONV_CG + threadIdx.x;
  const int d0 = cg * V;
  if (d0 >= Ek) return;
  const int t0 = blockIdx.y * CONV_TCH;
  const int t1 = min(L, t0 + CONV_TCH);
  const int b = blockIdx.z;
  auto row = [&](int t) -> const T* {
    return t < 0 ? cst + ((int64_t)b * (K - 1) + (K - 1) + t) * Ek + d0 : xz + ((int64_t)b * L + t) * ldxz + d0;
  };
  uint4 pf[CONV_PF];
#pragma unroll
  for (int i = 0; i < CONV_PF; ++i) pf[i] = (t0 + i < t1) ? *reinterpret_cast<const uint4*>(row(t0 + i)) : make_uint4(0, 0, 0, 0);
  float w[K][V], bias[V], win[K][V];
#pragma unroll
  for (int j = 0; j < K - 1; ++j) Vec<T, V>::load(row(t0 - (K - 1) + j), win[j + 1]);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    bias[v] = cb[d0 + v];
#pragma unroll
    for (int j = 0; j < K; ++j) w[j][v] = cw[(d0 + v) * K + j];
  }
  for (int t = t0; t < t1; t += CONV_PF) {
#pragma unroll
    for (int i = 0; i < CONV_PF; ++i) {
      if (t + i >= t1) break;
      const uint4 cur = pf[i];
      if (t + i + CONV_PF < t1) pf[i] = *reinterpret_cast<const uint4*>(row(t + i + CONV_PF));  // prefetch
#pragma unroll
      for (int j = 0; j < K - 1; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) win[j][v] = win[j + 1][v];
      if constexpr (sizeof(T) == 2) {
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&cur);
#pragma unroll
        for (int q = 0; q < V / 2; ++q) { const float2 f = __bfloat1622float2(h2[q]); win[K - 1][2 * q] = f.x; win[K - 1][2 * q + 1] = f.y; }
      } else {
        const float* f = reinterpret_cast<const float*>(&cur);
#pragma unroll
        for (int q = 0; q < V; ++q) win[K - 1][q] = f[q];
      }
      float o[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float acc = bias[v];
#pragma unroll
        for (int j = 0; j < K; ++j) acc = fmaf(w[j][v], win[j][v], acc);
        o[v] = FAST ? silu_tanh(acc) : silu<false>(acc);
      }
      Vec<T, V>::store(u + ((int64_t)b * L + t + i) * ldu + d0, o);
    }
  }
}

// bf16 prefill conv v3 (the launched one): persistent blocks, 2 per SM, walk work items (batch row,
// 1024-channel block, 16-token tile); the (16 + K - 1)-row input tile of the NEXT item is fetched by
// cp.async while the current one is convolved (double buffer), so each SM keeps ~76 KB in flight
// continuously instead of in one burst per block (v2: 254 us per Mamba-2.8B layer, 0.4 of HBM).
// A thread owns 8 channels x 8 tokens of a tile and stores 16-B vectors.
constexpr int C3_CH = 1024, C3_TT = 16, C3_THREADS = 256;
// Prefill conv1d + SiLU (row a2): persistent blocks (2 per SM) walk contiguous runs
// of 16-token x 1024-channel tiles of one channel block (taps kept in registers across the run); each
// tile (with its K - 1 halo rows) arrives by TMA -- four 256-channel boxes onto the buffer's mbarrier,
// double buffered -- and a sequence's first tile takes its halo from the cached window (166 -> 140 us
// per Mamba-2.8B layer against the cp.async version).
template <int K>
__global__ void __launch_bounds__(C3_THREADS, 2) conv1d_silu_v3_kernel(const __grid_constant__ CUtensorMap tm_x,
                                                                    const __nv_bfloat16* __restrict__ cst,
                                                                    const float* __restrict__ cw,
                                                                    const float* __restrict__ cb,
                                                                    __nv_bfloat16* __restrict__ u, int64_t ldu, int L,
                                                                    int Ek, int batch) {
  extern __shared__ __align__(128) __nv_bfloat16 sx3_raw[];
  __shared__ __align__(8) uint64_t mb[2];
  constexpr int ROWS = C3_TT + K - 1, CPR = C3_CH / 8, SUB = C3_CH / 256;
  // tile [SUB][ROWS][256]: one TMA box (256 channels x ROWS tokens) per sub-block
  auto sxp = [&](int buf, int r, int cgi) { return sx3_raw + ((buf * SUB + (cgi >> 5)) * ROWS + r) * 256 + (cgi & 31) * 8; };
  const int nchb = (Ek + C3_CH - 1) / C3_CH, ntt = (L + C3_TT - 1) / C3_TT;
  const int items = nchb * ntt * batch;
  const int tid = threadIdx.x, cg = tid % CPR, tl = tid / CPR;
  if (tid == 0) {
    tma_prefetch_desc(&tm_x);
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  auto coords = [&](int it, int& c0, int& t0, int& b) {
    t0 = (it % ntt) * C3_TT;
    const int r = it / ntt;
    c0 = (r % nchb) * C3_CH;
    b = r / nchb;
  };
  // thread 0: the tile's rows t0 - (K-1) .. t0 + C3_TT - 1 of this sequence's x (rows of the previous
  // sequence or below row 0 at t0 = 0 are replaced by the cached window after the load lands)
  auto load = [&](int buf, int it) {
    int c0, t0, b;
    coords(it, c0, t0, b);
    fence_proxy_async();  // the halo rows this buffer got from generic stores are overwritten by TMA
    mbar_arrive_expect_tx(&mb[buf], (uint32_t)(SUB * ROWS * 256 * 2));
    for (int j = 0; j < SUB; ++j)
      tma_load_2d(sx3_raw + (buf * SUB + j) * ROWS * 256, &tm_x, &mb[buf], c0 + 256 * j, b * L + t0 - (K - 1));
  };
  // a contiguous run of items per block (t-tiles fastest): the taps are reloaded only when the
  // channel block changes
  const int it0 = (int)((int64_t)items * blockIdx.x / gridDim.x), it1 = (int)((int64_t)items * (blockIdx.x + 1) / gridDim.x);
  int buf = 0, wc0 = -1;
  uint32_t ph = 0u;  // bit b: the parity buffer b waits for next
  float w[K][8], bias[8];
  if (tid == 0 && it0 < it1) load(0, it0);
  for (int it = it0; it < it1; ++it, buf ^= 1) {
    if (tid == 0 && it + 1 < it1) load(buf ^ 1, it + 1);
    int c0, t0, b;
    coords(it, c0, t0, b);
    const int d0 = c0 + cg * 8;
    if (c0 != wc0 && d0 < Ek) {
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        bias[v] = cb[d0 + v];
#pragma unroll
        for (int j = 0; j < K; ++j) w[j][v] = cw[(d0 + v) * K + j];
      }
    }
    wc0 = c0;
    mbar_wait(&mb[buf], (ph >> buf) & 1u);
    ph ^= 1u << buf;
    if (t0 == 0) {  // sequence start: the halo rows come from the cached window
      __syncthreads();
      for (int i = tid; i < (K - 1) * CPR; i += C3_THREADS) {
        const int r = i / CPR, cgi = i % CPR, ch = c0 + cgi * 8;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (ch < Ek) v = *reinterpret_cast<const uint4*>(cst + ((int64_t)b * (K - 1) + r) * Ek + ch);
        *reinterpret_cast<uint4*>(sxp(buf, r, cgi)) = v;
      }
      __syncthreads();
    }
    if (d0 < Ek) {
      constexpr int TPT = C3_TT / (C3_THREADS / CPR);  // tokens per thread
      const int tb = tl * TPT;
      float win[K][8];
#pragma unroll
      for (int j = 0; j < K - 1; ++j) Vec<__nv_bfloat16, 8>::load(sxp(buf, tb + j, cg), win[j + 1]);
#pragma unroll
      for (int i = 0; i < TPT; ++i) {
        const int t = t0 + tb + i;
        if (t >= L) break;
#pragma unroll
        for (int j = 0; j < K - 1; ++j)
#pragma unroll
          for (int v = 0; v < 8; ++v) win[j][v] = win[j + 1][v];
        Vec<__nv_bfloat16, 8>::load(sxp(buf, tb + i + K - 1, cg), win[K - 1]);
        float o[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          float acc = bias[v];
#pragma unroll
          for (int j = 0; j < K; ++j) acc = fmaf(w[j][v], win[j][v], acc);
          o[v] = silu_tanh(acc);
        }
        Vec<__nv_bfloat16, 8>::store(u + ((int64_t)b * L + t) * ldu + d0, o);
      }
    }
    __syncthreads();  // this buffer is refilled by the load issued in the next iteration
  }
}

// conv window after the chunk: last K-1 entries of xt = conv_state || x
template <typename T>
__global__ void conv_state_update_kernel(const T* __restrict__ xz, int64_t ldxz, T* __restrict__ cst, int batch,
                                         int L, int Ek, int K) {
  pdl_trigger();
  pdl_wait();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * Ek) return;
  const int b = idx / Ek, d = idx % Ek;
  float vals[8];
  for (int j = 0; j < K - 1; ++j) {
    const int p = L + j;  // position in xt
    vals[j] = (p < K - 1) ? io<T>::ld(cst + ((int64_t)b * (K - 1) + p) * Ek + d)
                          : io<T>::ld(xz + ((int64_t)b * L + (p - (K - 1))) * ldxz + d);
  }
  for (int j = 0; j < K - 1; ++j) io<T>::st(cst + ((int64_t)b * (K - 1) + j) * Ek + d, vals[j]);
}

// decode: one token, conv window shifted in place
template <typename T, bool FAST>
__global__ void conv_decode_kernel(const T* __restrict__ xz, int64_t ldxz, T* __restrict__ cst,
                                   const float* __restrict__ cw, const float* __restrict__ cb, T* __restrict__ u,
                                   int64_t ldu, int batch, int Ek, int K, float4* __restrict__ z0, int64_t n0,
                                   float4* __restrict__ z1, int64_t n1, float* __restrict__ xacc) {
  pdl_trigger();
  pdl_wait();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  // zero the split-K accumulation targets of the following GEMMs (x_proj, out_proj partial)
  for (int64_t i = idx; i < n0; i += (int64_t)gridDim.x * blockDim.x) z0[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = idx; i < n1; i += (int64_t)gridDim.x * blockDim.x) z1[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (idx >= batch * Ek) return;
  const int b = idx / Ek, d = idx % Ek;
  float win[8];
  for (int j = 0; j < K - 1; ++j) win[j] = io<T>::ld(cst + ((int64_t)b * (K - 1) + j) * Ek + d);
  if (xacc) {  // x from the decode in_proj fp32 accumulator; this thread is its only reader -> re-zero
    float* p = xacc + (int64_t)b * ldxz + d;
    win[K - 1] = *p;
    *p = 0.f;
  } else {
    win[K - 1] = io<T>::ld(xz + (int64_t)b * ldxz + d);
  }
  float acc = cb[d];
  for (int j = 0; j < K; ++j) acc = fmaf(cw[d * K + j], win[j], acc);
  io<T>::st(u + (int64_t)b * ldu + d, silu<FAST>(acc));
  for (int j = 0; j < K - 1; ++j) io<T>::st(cst + ((int64_t)b * (K - 1) + j) * Ek + d, win[j + 1]);
}

// ---------------------------------------------------------------- unpack (AR#1 consumer)
constexpr int kMaxP = 320;  // R + 2N <= 320
template <typename T>
__global__ void __launch_bounds__(256) unpack_kernel(Peers src, int nsrc, int64_t off, int M, int hloc, int R, int N,
                                                     int rmsnorm, float eps, T* __restrict__ dlow,
                                                     float* __restrict__ BC) {
  pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= M * hloc) return;
  const int m = warp / hloc, hd = warp % hloc;
  const int P = R + 2 * N;
  const int64_t base = (int64_t)m * hloc * P + (int64_t)hd * P;
  constexpr int CPL = kMaxP / 32;
  float v[CPL];
  float ss[3] = {0.f, 0.f, 0.f};
  // fixed rank order 0..nsrc-1 (reading Q12): every load of a source issued before any add, so a row's
  // loads are in flight together (a per-element source loop serialised them: latency-bound)
  {
    const float* s0 = reinterpret_cast<const float*>(reinterpret_cast<const char*>(src.p[0]) + off) + base;
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = lane + 32 * i;
      v[i] = c < P ? s0[c] : 0.f;
    }
  }
  for (int sr = 1; sr < nsrc; ++sr) {
    const float* sp = reinterpret_cast<const float*>(reinterpret_cast<const char*>(src.p[sr]) + off) + base;
    float t[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) t[i] = lane + 32 * i < P ? sp[lane + 32 * i] : 0.f;
#pragma unroll
    for (int i = 0; i < CPL; ++i) v[i] = v[i] + t[i];
  }
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int c = lane + 32 * i;
    if (c < P) {
      const int f = c < R ? 0 : (c < R + N ? 1 : 2);
      ss[f] = fmaf(v[i], v[i], ss[f]);
    }
  }
  float scale[3] = {1.f, 1.f, 1.f};
  if (rmsnorm) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      float x = ss[f];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      const int cnt = f == 0 ? R : N;
      scale[f] = 1.0f / sqrtf(x / (float)cnt + eps);
    }
  }
  T* dl = dlow + ((int64_t)hd * M + m) * R;
  float* bc = BC + ((int64_t)hd * M + m) * 2 * N;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int c = lane + 32 * i;
    if (c < R)
      io<T>::st(dl + c, v[i] * scale[0]);
    else if (c < R + N)
      bc[c - R] = v[i] * scale[1];
    else if (c < P)
      bc[c - R] = v[i] * scale[2];
  }
}

// 2^x for x <= 0 on the FMA pipe (packed fp32x2): round-to-nearest split by the 1.5 * 2^23 magic
// number, degree-5 polynomial for 2^f on [-0.5, 0.5] (max rel. error 2.6e-7), exponent added in the
// integer pipe
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = fadd2(x, magic);
  const float2 jf = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(jf, make_float2(-1.f, -1.f), x);
  float2 p = ffma2(f, make_float2(0.00132764654699713f, 0.00132764654699713f),
                   make_float2(0.009675541892647743f, 0.009675541892647743f));
  p = ffma2(p, f, make_float2(0.05550713464617729f, 0.05550713464617729f));
  p = ffma2(p, f, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = ffma2(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = ffma2(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// ---------------------------------------------------------------- selective scan (prefill)

constexpr int SC_THREADS = 128;  // channels per block

// One thread per (batch row, channel); N states in registers; tiles of u, delta, z (bf16 or
// fp32: SC_TT tokens x 128 channels) and B||C (fp32: SC_TT tokens x 2N) staged through shared
// memory by TMA (cp.async.bulk.tensor 2D boxes, one thread issues the tile's four loads onto the
// buffer's mbarrier), double buffered.  h_t = exp(delta A) h_{t-1} + delta B_t u_t;
// y = <C_t, h_t> + D u;  g = y SiLU(z).  The tensor maps span all batch * L token rows, so a tile's
// rows past this row's L belong to the next batch row (loaded, never used) or lie outside the
// tensor (zero-filled); channels past nch are zero-filled.
template <typename T, int N, bool FAST>
__global__ void __launch_bounds__(SC_THREADS) scan_kernel(const __grid_constant__ CUtensorMap tm_u,
                                                          const __grid_constant__ CUtensorMap tm_d,
                                                          const __grid_constant__ CUtensorMap tm_z,
                                                          const __grid_constant__ CUtensorMap tm_bc,
                                                          const float* __restrict__ a_log,
                                                          const float* __restrict__ d_skip, float* __restrict__ h,
                                                          int64_t h_bstride, T* __restrict__ g, int64_t ldg, int L,
                                                          int nch) {
  constexpr int SC_TT = sizeof(T) == 2 ? 16 : 8;  // tokens per staged tile (static smem < 48 KB)
  __shared__ __align__(128) T su[2][SC_TT][SC_THREADS];
  __shared__ __align__(128) T sd[2][SC_TT][SC_THREADS];
  __shared__ __align__(128) T sz[2][SC_TT][SC_THREADS];
  __shared__ __align__(128) float sbc[2][SC_TT][2 * N];
  __shared__ __align__(8) uint64_t mb[2];
  constexpr uint32_t kTileBytes = 3u * SC_TT * SC_THREADS * sizeof(T) + SC_TT * 2 * N * 4;

  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const int cbase = blockIdx.x * SC_THREADS;
  const int d = cbase + tid;
  const bool valid = d < nch;
  const int64_t row0 = (int64_t)b * L;
  if (tid == 0) {
    tma_prefetch_desc(&tm_u);
    tma_prefetch_desc(&tm_d);
    tma_prefetch_desc(&tm_z);
    tma_prefetch_desc(&tm_bc);
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();

  auto load_tile = [&](int buf, int tile) {  // thread 0
    const int row = (int)(row0 + tile * SC_TT);
    mbar_arrive_expect_tx(&mb[buf], kTileBytes);
    tma_load_2d(&su[buf][0][0], &tm_u, &mb[buf], cbase, row);
    tma_load_2d(&sd[buf][0][0], &tm_d, &mb[buf], cbase, row);
    tma_load_2d(&sz[buf][0][0], &tm_z, &mb[buf], cbase, row);
    tma_load_2d(&sbc[buf][0][0], &tm_bc, &mb[buf], 0, row);
  };

  float A[N], hs[N];
  float2 A2[N / 2], h2[N / 2];
  float Dd = 0.f;
  float* hp = h + (int64_t)b * h_bstride + (int64_t)(valid ? d : 0) * N;
  if (valid) {
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float a = -expf(a_log[(int64_t)d * N + n]);
      A[n] = FAST ? a * 1.4426950408889634f : a;
      hs[n] = hp[n];
    }
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      A2[i] = make_float2(A[2 * i], A[2 * i + 1]);
      h2[i] = make_float2(hs[2 * i], hs[2 * i + 1]);
    }
    Dd = d_skip[d];
  }

  const int ntiles = (L + SC_TT - 1) / SC_TT;
  if (tid == 0) load_tile(0, 0);
  for (int it = 0; it < ntiles; ++it) {
    const int buf = it & 1;
    // the other buffer was released by every thread at the end of the previous tile
    if (tid == 0 && it + 1 < ntiles) load_tile(buf ^ 1, it + 1);
    mbar_wait(&mb[buf], (uint32_t)(it >> 1) & 1u);
    if (valid) {
      const int tb = it * SC_TT;
      const int tn = min(SC_TT, L - tb);
      if constexpr (FAST) {
        // packed fp32x2 state math: 16 ex2 on the MUFU pipe, 32 FFMA2/FMUL2 on the FMA pipe per token
        for (int r = 0; r < tn; ++r) {
          const float uu = io<T>::ld(&su[buf][r][tid]);
          const float de = io<T>::ld(&sd[buf][r][tid]);
          const float zz = io<T>::ld(&sz[buf][r][tid]);
          const float2 de2 = make_float2(de, de);
          const float du = de * uu;
          const float2 du2 = make_float2(du, du);
          const float4* B4 = reinterpret_cast<const float4*>(sbc[buf][r]);
          const float4* C4 = reinterpret_cast<const float4*>(sbc[buf][r] + N);
          float2 ya = make_float2(0.f, 0.f), yb = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < N / 4; ++q) {
            const float4 b4 = B4[q], c4 = C4[q];
            const float2 dA0 = fmul2(de2, A2[2 * q]);
            const float2 dA1 = fmul2(de2, A2[2 * q + 1]);
            const float2 a0 = make_float2(ex2_approx(dA0.x), ex2_approx(dA0.y));
            // the last pair of states on the FMA pipe (the kernel is MUFU-bound: 883 vs 894 us per
            // Mamba-2.8B layer; four states there measured 959 us)
            const float2 a1 = q == N / 4 - 1 ? exp2_poly2(dA1) : make_float2(ex2_approx(dA1.x), ex2_approx(dA1.y));
            h2[2 * q] = ffma2(a0, h2[2 * q], fmul2(du2, make_float2(b4.x, b4.y)));
            h2[2 * q + 1] = ffma2(a1, h2[2 * q + 1], fmul2(du2, make_float2(b4.z, b4.w)));
            ya = ffma2(make_float2(c4.x, c4.y), h2[2 * q], ya);
            yb = ffma2(make_float2(c4.z, c4.w), h2[2 * q + 1], yb);
          }
          float y = (ya.x + ya.y) + (yb.x + yb.y);
          y = fmaf(Dd, uu, y);
          io<T>::st(g + (row0 + tb + r) * ldg + d, y * silu_tanh(zz));
        }
      } else {
        for (int r = 0; r < tn; ++r) {
          const float uu = io<T>::ld(&su[buf][r][tid]);
          const float de = io<T>::ld(&sd[buf][r][tid]);
          const float zz = io<T>::ld(&sz[buf][r][tid]);
          const float du = de * uu;
          const float* Bt = sbc[buf][r];
          const float* Ct = Bt + N;
          float y = 0.f;
#pragma unroll
          for (int n = 0; n < N; ++n) {
            const float a = expf(de * A[n]);
            hs[n] = fmaf(a, hs[n], du * Bt[n]);
            y = fmaf(Ct[n], hs[n], y);
          }
          y = fmaf(Dd, uu, y);
          io<T>::st(g + (row0 + tb + r) * ldg + d, y * silu<false>(zz));
        }
      }
    }
    __syncthreads();
  }
  if (valid) {
    if constexpr (FAST) {
#pragma unroll
      for (int i = 0; i < N / 2; ++i) { hs[2 * i] = h2[i].x; hs[2 * i + 1] = h2[i].y; }
    }
#pragma unroll
    for (int n = 0; n < N; ++n) hp[n] = hs[n];
  }
}

// ---------------------------------------------------------------- decode step
// Body in dstep.cuh (shared with the out_proj GEMM, which can run it as its B-operand producer).
// one (batch row, channel) item per thread: 640 blocks of 128 threads for Mamba-2.8B at batch 16 (a
// 4-row-per-thread variant, 160 blocks with 4x fewer W_dt reads, and a 2-row one measured slower)
template <typename T, int N, bool FAST, int IPT = 1>
__global__ void __launch_bounds__(DS_THREADS, 5) decode_step_kernel(DStepArgs a, Peers src, int nsrc) {
  extern __shared__ __align__(16) float dsm[];
  pdl_trigger();
  dstep_unit<T, N, FAST, DS_THREADS, IPT>(a, src, nsrc, blockIdx.x * DS_CH, blockIdx.y * DS_BB * IPT, threadIdx.x,
                                            dsm, -1, true);
}
// ---------------------------------------------------------------- RMSNorm (glue)
// One 128-thread block per row, the row cached in registers (<= 16 float4 per thread).
template <typename T>
__global__ void __launch_bounds__(128) rmsnorm_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                      float eps, T* __restrict__ y, int64_t M, int D) {
  pdl_trigger();
  pdl_wait();
  constexpr int MAXV = 16;
  __shared__ float red[4];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + row * D);
  const int nv = D / 4;
  float4 v[MAXV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int k = tid + i * 128;
    if (k < nv) {
      v[i] = xr[k];
      ss = fmaf(v[i].x, v[i].x, ss); ss = fmaf(v[i].y, v[i].y, ss);
      ss = fmaf(v[i].z, v[i].z, ss); ss = fmaf(v[i].w, v[i].w, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  const float tot = (red[0] + red[1]) + (red[2] + red[3]);
  const float rs = 1.0f / sqrtf(tot / (float)D + eps);
  T* yr = y + row * D;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int k = tid + i * 128;
    if (k < nv) {
      float4 ww = make_float4(1.f, 1.f, 1.f, 1.f);
      if (w) ww = reinterpret_cast<const float4*>(w)[k];
      if constexpr (sizeof(T) == 2) {  // one 8-B store of 4 bf16
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * rs * ww.x, v[i].y * rs * ww.y);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * rs * ww.z, v[i].w * rs * ww.w);
        uint2 pk;
        pk.x = *reinterpret_cast<const uint32_t*>(&lo);
        pk.y = *reinterpret_cast<const uint32_t*>(&hi);
        reinterpret_cast<uint2*>(yr)[k] = pk;
      } else {
        io<T>::st(yr + 4 * k, v[i].x * rs * ww.x);
        io<T>::st(yr + 4 * k + 1, v[i].y * rs * ww.y);
        io<T>::st(yr + 4 * k + 2, v[i].z * rs * ww.z);
        io<T>::st(yr + 4 * k + 3, v[i].w * rs * ww.w);
      }
    }
  }
}

// ---------------------------------------------------------------- int8 quantise / reduce
// One warp per block of blk = 32*VPL values: amax, s = amax/127 (IEEE), q = rint(o/s) in [-127,127].
template <int VPL>
__global__ void quantize_kernel(const float* __restrict__ x, int64_t nblocks, int8_t* __restrict__ q,
                                float* __restrict__ scale) {
  pdl_trigger();
  pdl_wait();
  const int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (blk >= nblocks) return;
  const float* xb = x + blk * 32 * VPL + lane * VPL;
  float v[VPL];
  float am = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    v[i] = xb[i];
    am = fmaxf(am, fabsf(v[i]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  const float s = __fdiv_rn(am, 127.0f);
  int8_t* qb = q + blk * 32 * VPL + lane * VPL;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    int c = 0;
    if (s != 0.f) {
      c = __float2int_rn(__fdiv_rn(v[i], s));
      c = max(-127, min(127, c));
    }
    qb[i] = (int8_t)c;
  }
  if (lane == 0) scale[blk] = s;
}

// Optional next-layer pre-norm statistics of the updated residual rows (RowOut, reading Q22 at TP > 1):
// 16 consecutive values v of element group i (row m = 16 i / D) -> cpy = bf16(v) and, per 32-column chunk
// (groups i, i ^ 1), its sum of squares -> ssq[m * D/32 + chunk] (the finalize kernel sums the chunks of
// a row in fixed order, as after the TP = 1 out_proj epilogue).  Every rank runs the same arithmetic on
// the same bits, so the replicas stay equal.
struct RowOut {
  __nv_bfloat16* cpy;
  float* ssq;
  int D;
};
SSM_DEV void rowout16(const RowOut& ro, int64_t i, const float (&v)[16]) {
  uint32_t pk[8];
  float sq = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    __nv_bfloat162 t2 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    pk[j] = *reinterpret_cast<uint32_t*>(&t2);
    sq = fmaf(v[2 * j], v[2 * j], sq);
    sq = fmaf(v[2 * j + 1], v[2 * j + 1], sq);
  }
  uint4* c = reinterpret_cast<uint4*>(ro.cpy + i * 16);
  c[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  c[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  // the partner group of the chunk is active whenever this one is (n16 even)
  sq += __shfl_xor_sync(__activemask(), sq, 1);
  if ((i & 1) == 0) {
    const int64_t e0 = i * 16;
    ro.ssq[(e0 / ro.D) * (ro.D / 32) + (e0 % ro.D) / 32] = sq;
  }
}

__global__ void qar_reduce_kernel(Peers src, int k, int64_t q_off, int64_t s_off, int64_t n16, int blk,
                                  float* __restrict__ out, int accumulate, RowOut ro) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n16) return;
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0.f;
  const int64_t sidx = (i * 16) / blk;
  for (int r = 0; r < k; ++r) {  // fixed rank order 0..k-1: bitwise-identical on every rank
    const char* base = reinterpret_cast<const char*>(src.p[r]);
    const int4 qv = *reinterpret_cast<const int4*>(base + q_off + i * 16);
    const float s = reinterpret_cast<const float*>(base + s_off)[sidx];
    const int8_t* qq = reinterpret_cast<const int8_t*>(&qv);
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fmaf(s, (float)qq[j], acc[j]);
  }
  float4* o = reinterpret_cast<float4*>(out + i * 16);
  float fin[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 v = accumulate ? o[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    v.x += acc[4 * q]; v.y += acc[4 * q + 1]; v.z += acc[4 * q + 2]; v.w += acc[4 * q + 3];
    o[q] = v;
    fin[4 * q] = v.x; fin[4 * q + 1] = v.y; fin[4 * q + 2] = v.z; fin[4 * q + 3] = v.w;
  }
  if (ro.cpy) rowout16(ro, i, fin);
}

__global__ void f32_reduce_kernel(Peers src, int k, int64_t off, int64_t n4, float* __restrict__ out, int accumulate) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 acc = reinterpret_cast<const float4*>(reinterpret_cast<const char*>(src.p[0]) + off)[i];
  for (int r = 1; r < k; ++r) {
    const float4 v = reinterpret_cast<const float4*>(reinterpret_cast<const char*>(src.p[r]) + off)[i];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  float4* o = reinterpret_cast<float4*>(out) + i;
  if (accumulate) {
    float4 v = *o;
    acc.x = v.x + acc.x; acc.y = v.y + acc.y; acc.z = v.z + acc.z; acc.w = v.w + acc.w;
  }
  *o = acc;
}

// ---------------------------------------------------------------- two-shot int8 all-reduce (reading Q6)
// Shared per-block scales, so codes of different ranks add exactly:
//   (1) amax_r[b] -> own buffer; barrier
//   (2) s[b] = fl32(max_r amax_r[b] / 127); q_r = clamp(rint(fl32(o_r / s)), +-127) -> own buffer; barrier
//   (3) reduce-scatter: rank j sums the k codes of its shard exactly (int16, |sum| <= 127 k); barrier
//   (4) all-gather: out[i] (+)= fl32(s[b] * sum_j[i]) read from the shard's owner.
// Wire per rank: (k-1)/k n B of int8 codes + (k-1)/k 2n B of int16 sums (+ scales) vs (k-1) n B
// one-shot.  Error <= k s / 2 <= k max_r amax_r / 254 per element (the north_star bound).
template <int VPL>
__global__ void amax_kernel(const float* __restrict__ x, int64_t nblocks, float* __restrict__ amax) {
  pdl_trigger();
  pdl_wait();
  const int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (blk >= nblocks) return;
  const float* xb = x + blk * 32 * VPL + lane * VPL;
  float am = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) am = fmaxf(am, fabsf(xb[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  if (lane == 0) amax[blk] = am;
}

template <int VPL>
__global__ void quant_shared_kernel(const float* __restrict__ x, int64_t nblocks, Peers src, int k, int64_t amax_off,
                                    int8_t* __restrict__ q, float* __restrict__ scale) {
  pdl_trigger();
  pdl_wait();
  const int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (blk >= nblocks) return;
  float A = 0.f;
  for (int r = 0; r < k; ++r)
    A = fmaxf(A, reinterpret_cast<const float*>(reinterpret_cast<const char*>(src.p[r]) + amax_off)[blk]);
  const float s = __fdiv_rn(A, 127.0f);
  const float* xb = x + blk * 32 * VPL + lane * VPL;
  int8_t* qb = q + blk * 32 * VPL + lane * VPL;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    int c = 0;
    if (s != 0.f) c = max(-127, min(127, __float2int_rn(__fdiv_rn(xb[i], s))));
    qb[i] = (int8_t)c;
  }
  if (lane == 0) scale[blk] = s;
}

__global__ void rs16_kernel(Peers src, int k, int64_t q_off, int64_t lo, int64_t n16, int16_t* __restrict__ sums) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // 16-element group of this rank's shard
  if (i >= n16) return;
  int acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0;
  for (int r = 0; r < k; ++r) {
    const int4 qv = *reinterpret_cast<const int4*>(reinterpret_cast<const char*>(src.p[r]) + q_off + lo + i * 16);
    const int8_t* qq = reinterpret_cast<const int8_t*>(&qv);
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] += qq[j];
  }
  int16_t o[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = (int16_t)acc[j];
  reinterpret_cast<int4*>(sums + i * 16)[0] = reinterpret_cast<const int4*>(o)[0];
  reinterpret_cast<int4*>(sums + i * 16)[1] = reinterpret_cast<const int4*>(o)[1];
}

__global__ void ag16_kernel(Peers src, int64_t sum_off, int64_t shard, int64_t n16, const float* __restrict__ scale,
                            int blk, float* __restrict__ out, int accumulate, RowOut ro) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n16) return;
  const int64_t e0 = i * 16;
  const int j = (int)(e0 / shard);  // owner of this 16-element group (shard % 16 == 0)
  const int16_t* sp = reinterpret_cast<const int16_t*>(reinterpret_cast<const char*>(src.p[j]) + sum_off) + (e0 - (int64_t)j * shard);
  int16_t qv[16];
  reinterpret_cast<int4*>(qv)[0] = reinterpret_cast<const int4*>(sp)[0];
  reinterpret_cast<int4*>(qv)[1] = reinterpret_cast<const int4*>(sp)[1];
  const float s = scale[e0 / blk];  // blk % 16 == 0: one block per group
  float4* o = reinterpret_cast<float4*>(out + e0);
  float fin[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 v = accumulate ? o[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    // fl32(s * Q) then an fp32 add, as the oracle rounds (no fma contraction)
    v.x = __fadd_rn(v.x, __fmul_rn(s, (float)qv[4 * q])); v.y = __fadd_rn(v.y, __fmul_rn(s, (float)qv[4 * q + 1]));
    v.z = __fadd_rn(v.z, __fmul_rn(s, (float)qv[4 * q + 2])); v.w = __fadd_rn(v.w, __fmul_rn(s, (float)qv[4 * q + 3]));
    o[q] = v;
    fin[4 * q] = v.x; fin[4 * q + 1] = v.y; fin[4 * q + 2] = v.z; fin[4 * q + 3] = v.w;
  }
  if (ro.cpy) rowout16(ro, i, fin);
}

// ---------------------------------------------------------------- requantised two-shot int8 (labelled variant)
// Stage 2 (shard owner): S = fl32 sum over ranks (fixed order) of fl32(s_r q_r), then per-block
// requantisation (amax, s' = fl32(amax / 127), q' = clamp(rint(fl32(S / s')))) -- the operations of
// qar_ref.qallreduce_requant.  One warp per block of blk = 32 VPL elements of this rank's shard.
template <int VPL>
__global__ void rq_reduce_kernel(Peers src, int k, int64_t q_off, int64_t s_off, int64_t lo, int64_t nb_shard,
                                 int8_t* __restrict__ q2, float* __restrict__ s2) {
  pdl_trigger();
  pdl_wait();
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= nb_shard) return;
  constexpr int blk = 32 * VPL;
  const int64_t e0 = lo + b * blk + lane * VPL, gb = lo / blk + b;
  float acc[VPL];
  for (int r = 0; r < k; ++r) {  // fixed rank order 0..k-1
    const char* base = reinterpret_cast<const char*>(src.p[r]);
    const float sr = reinterpret_cast<const float*>(base + s_off)[gb];
    const int8_t* qr = reinterpret_cast<const int8_t*>(base + q_off) + e0;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const float d = __fmul_rn(sr, (float)qr[i]);
      acc[i] = r == 0 ? d : __fadd_rn(acc[i], d);
    }
  }
  float am = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) am = fmaxf(am, fabsf(acc[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  const float sp = __fdiv_rn(am, 127.0f);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    int c = 0;
    if (sp != 0.f) c = max(-127, min(127, __float2int_rn(__fdiv_rn(acc[i], sp))));
    q2[b * blk + lane * VPL + i] = (int8_t)c;
  }
  if (lane == 0) s2[b] = sp;
}

// Stage 3 (all-gather): out[i] (+)= fl32(s'_o q'_o[i]) from the shard owner o = i / shard.
__global__ void rq_gather_kernel(Peers src, int64_t q2_off, int64_t s2_off, int64_t shard, int64_t n16, int blk,
                                 float* __restrict__ out, int accumulate) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n16) return;
  const int64_t e0 = i * 16;
  const int o = (int)(e0 / shard);
  const char* base = reinterpret_cast<const char*>(src.p[o]);
  const int64_t le = e0 - (int64_t)o * shard;
  const int4 qv = *reinterpret_cast<const int4*>(base + q2_off + le);
  const int8_t* qq = reinterpret_cast<const int8_t*>(&qv);
  const float sp = reinterpret_cast<const float*>(base + s2_off)[le / blk];
  float4* dst = reinterpret_cast<float4*>(out + e0);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 v = accumulate ? dst[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    v.x = __fadd_rn(v.x, __fmul_rn(sp, (float)qq[4 * q])); v.y = __fadd_rn(v.y, __fmul_rn(sp, (float)qq[4 * q + 1]));
    v.z = __fadd_rn(v.z, __fmul_rn(sp, (float)qq[4 * q + 2])); v.w = __fadd_rn(v.w, __fmul_rn(sp, (float)qq[4 * q + 3]));
    dst[q] = v;
  }
}

// ---------------------------------------------------------------- 16-bit-wire all-reduces
// fp16 (the paper's FP32 -> FP16 wire) and bf16 (the custom bf16 arm, SURVEY.md
// §8(d)): cast 8 fp32 -> 8 16-bit values per thread (cvt.rn: IEEE round-to-nearest-even; fp16
// overflow -> inf), exchanged one-shot, then summed in fp32.
template <typename H> struct Wire16;
template <> struct Wire16<__half> {
  SSM_DEV static uint32_t pack(float a, float b) { __half2 h = __floats2half2_rn(a, b); return *reinterpret_cast<uint32_t*>(&h); }
  SSM_DEV static float2 unpack(uint32_t w) { return __half22float2(*reinterpret_cast<const __half2*>(&w)); }
};
template <> struct Wire16<__nv_bfloat16> {
  SSM_DEV static uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  SSM_DEV static float2 unpack(uint32_t w) { return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w)); }
};
template <typename H>
__global__ void w16_cast_kernel(const float* __restrict__ x, int64_t n8, uint4* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const float4 a = reinterpret_cast<const float4*>(x)[2 * i];
  const float4 b = reinterpret_cast<const float4*>(x)[2 * i + 1];
  out[i] = make_uint4(Wire16<H>::pack(a.x, a.y), Wire16<H>::pack(a.z, a.w), Wire16<H>::pack(b.x, b.y),
                      Wire16<H>::pack(b.z, b.w));
}
// Reduce: acc = fl32(h_0); acc = acc + fl32(h_r) for r = 1..k-1 (fixed order: bitwise-identical
// replicas, Q12); out = out + acc (accumulate) or acc.
template <typename H>
__global__ void w16_reduce_kernel(Peers src, int k, int64_t off, int64_t n8, float* __restrict__ out, int accumulate) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  float acc[8];
  for (int r = 0; r < k; ++r) {
    const uint4 raw = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(src.p[r]) + off)[i];
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = Wire16<H>::unpack(w[j]);
      if (r == 0) { acc[2 * j] = f.x; acc[2 * j + 1] = f.y; }
      else { acc[2 * j] = acc[2 * j] + f.x; acc[2 * j + 1] = acc[2 * j + 1] + f.y; }
    }
  }
  float4* o = reinterpret_cast<float4*>(out) + 2 * i;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    float4 v = accumulate ? o[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    v.x = v.x + acc[4 * q]; v.y = v.y + acc[4 * q + 1]; v.z = v.z + acc[4 * q + 2]; v.w = v.w + acc[4 * q + 3];
    o[q] = v;
  }
}

// ---------------------------------------------------------------- cross-rank barrier
// Signal area at the head of every symmetric buffer: uint32 slot[8] (slot[p] = last epoch
// rank p announced to us), uint32 error word at +64 B, uint32 epoch counter at +128 B.
// The epoch lives in device memory so a captured CUDA graph advances it on every replay
// (every rank executes the same barrier sequence, so the counters agree).
__global__ void peer_barrier_kernel(Peers bufs, int rank, int k) {
  pdl_trigger();
  pdl_wait();
  __shared__ uint32_t s_epoch;
  const int t = threadIdx.x;
  uint32_t* own = reinterpret_cast<uint32_t*>(bufs.p[rank]);
  if (t == 0) s_epoch = atomicAdd(own + 32, 1u) + 1u;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  if (t < k) {
    fence_sys();
    st_release_sys(reinterpret_cast<uint32_t*>(bufs.p[t]) + rank, epoch);
  }
  __syncwarp();
  if (t < k) {
    const uint32_t* slot = own + t;
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(slot) - epoch) < 0) {
      if (globaltimer() - t0 > 20ull * 1000000000ull) {
        atomicExch(own + 16, 1u);
        break;
      }
    }
  }
  __syncwarp();
  fence_sys();
}

template <typename T, bool F>
cudaError_t conv_dispatch(const void* xz, int64_t ldxz, const void* cs, const float* cw, const float* cb, void* u,
                          int64_t ldu, int batch, int L, int Ek, int K, cudaStream_t s) {
  if constexpr (sizeof(T) == 2 && F) {
    if (Ek % 8 == 0 && ldxz % 8 == 0 && ldu % 8 == 0) {  // persistent smem-pipelined kernel (bf16)
      const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(xz);
      const __nv_bfloat16* c = reinterpret_cast<const __nv_bfloat16*>(cs);
      __nv_bfloat16* uu = reinterpret_cast<__nv_bfloat16*>(u);
      if (K < 2 || K > 4) return cudaErrorInvalidValue;
      const size_t sm = (size_t)2 * (C3_TT + K - 1) * C3_CH * 2;
      static bool attr[5] = {false, false, false, false, false};
      const void* fn = K == 2 ? (const void*)conv1d_silu_v3_kernel<2> : K == 3 ? (const void*)conv1d_silu_v3_kernel<3>
                                                                             : (const void*)conv1d_silu_v3_kernel<4>;
      cudaError_t e_ = cudaSuccess;
      if (!attr[K]) {
        e_ = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e_ != cudaSuccess) return e_;
        attr[K] = true;
      }
      static int sms = 0;
      if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      }
      const int items = ((Ek + C3_CH - 1) / C3_CH) * ((L + C3_TT - 1) / C3_TT) * batch;
      const int grid3 = items < 2 * sms ? items : 2 * sms;
      CUtensorMap mx;
      if ((int64_t)batch * L > INT32_MAX || !encode_tmap_2d(&mx, x, (int64_t)batch * L, Ek, ldxz, 2, 256, C3_TT + K - 1))
        return cudaErrorInvalidValue;
      switch (K) {
        case 2: e_ = launch(conv1d_silu_v3_kernel<2>, grid3, C3_THREADS, sm, s, mx, c, cw, cb, uu, ldu, L, Ek, batch); break;
        case 3: e_ = launch(conv1d_silu_v3_kernel<3>, grid3, C3_THREADS, sm, s, mx, c, cw, cb, uu, ldu, L, Ek, batch); break;
        default: e_ = launch(conv1d_silu_v3_kernel<4>, grid3, C3_THREADS, sm, s, mx, c, cw, cb, uu, ldu, L, Ek, batch); break;
      }
      if (e_ != cudaSuccess) return e_;
      return cudaGetLastError();
    }
  }
  constexpr int V = vec_of<T>();
  dim3 grid((Ek / V + CONV_CG - 1) / CONV_CG, (L + CONV_TCH - 1) / CONV_TCH, batch);
  const T* x = reinterpret_cast<const T*>(xz);
  const T* c = reinterpret_cast<const T*>(cs);
  T* uu = reinterpret_cast<T*>(u);
  constexpr int NT = CONV_CG;
  switch (K) {
    case 2: { cudaError_t e_ = launch(conv1d_silu_kernel<T, 2, F>, grid, NT, 0, s, x, ldxz, c, cw, cb, uu, ldu, L, Ek); if (e_ != cudaSuccess) return e_; } break;
    case 3: { cudaError_t e_ = launch(conv1d_silu_kernel<T, 3, F>, grid, NT, 0, s, x, ldxz, c, cw, cb, uu, ldu, L, Ek); if (e_ != cudaSuccess) return e_; } break;
    case 4: { cudaError_t e_ = launch(conv1d_silu_kernel<T, 4, F>, grid, NT, 0, s, x, ldxz, c, cw, cb, uu, ldu, L, Ek); if (e_ != cudaSuccess) return e_; } break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Pre-norm statistic without the normalisation (prefill with the norm folded into the in_proj, reading
// Q22): y = bf16(x) and ss[row] = sum_d x[row][d]^2, one block per row, the same fixed reduction
// order as rmsnorm_kernel.
__global__ void __launch_bounds__(128) rowstats_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                                       float* __restrict__ ss, int64_t M, int D) {
  pdl_trigger();
  pdl_wait();
  constexpr int MAXV = 16;
  __shared__ float red[4];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + row * D);
  const int nv = D / 4;
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int k = tid + i * 128;
    if (k < nv) {
      const float4 v = xr[k];
      acc = fmaf(v.x, v.x, acc); acc = fmaf(v.y, v.y, acc);
      acc = fmaf(v.z, v.z, acc); acc = fmaf(v.w, v.w, acc);
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
      uint2 pk;
      pk.x = *reinterpret_cast<const uint32_t*>(&lo);
      pk.y = *reinterpret_cast<const uint32_t*>(&hi);
      reinterpret_cast<uint2*>(y + row * D)[k] = pk;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) ss[row] = (red[0] + red[1]) + (red[2] + red[3]);
}

// ss[m] = the row's per-32-column partial sums of squares (written by the out_proj epilogue, Epilogue::ssq)
// summed in a fixed order: one warp per row, lanes stride the partials, then a shuffle tree.
__global__ void __launch_bounds__(256) ssq_finalize_kernel(const float* __restrict__ part, int nchunk,
                                                           float* __restrict__ ss, int64_t M) {
  pdl_trigger();
  pdl_wait();
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  float acc = 0.f;
  for (int c = lane; c < nchunk; c += 32) acc += part[row * nchunk + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) ss[row] = acc;
}

}  // namespace

// ==================================================================== launchers
cudaError_t launch_conv1d_silu(int bf16, const void* xz, int64_t ldxz, const void* cs, const float* cw,
                               const float* cb, void* u, int64_t ldu, int batch, int L, int Ek, int K,
                               cudaStream_t s) {
  if (batch <= 0 || L <= 0) return cudaSuccess;
  if (bf16) return conv_dispatch<__nv_bfloat16, true>(xz, ldxz, cs, cw, cb, u, ldu, batch, L, Ek, K, s);
  return conv_dispatch<float, false>(xz, ldxz, cs, cw, cb, u, ldu, batch, L, Ek, K, s);
}

cudaError_t launch_conv_state_update(int bf16, const void* xz, int64_t ldxz, void* cs, int batch, int L, int Ek,
                                     int K, cudaStream_t s) {
  const int n = batch * Ek;
  if (n <= 0 || L <= 0) return cudaSuccess;
  if (bf16)
    { cudaError_t e_ = launch(conv_state_update_kernel<__nv_bfloat16>, (n + 255) / 256, 256, 0, s, 
        reinterpret_cast<const __nv_bfloat16*>(xz), ldxz, reinterpret_cast<__nv_bfloat16*>(cs), batch, L, Ek, K); if (e_ != cudaSuccess) return e_; }
  else
    { cudaError_t e_ = launch(conv_state_update_kernel<float>, (n + 255) / 256, 256, 0, s, reinterpret_cast<const float*>(xz), ldxz,
                                                                     reinterpret_cast<float*>(cs), batch, L, Ek, K); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

cudaError_t launch_conv_decode(int bf16, const void* xz, int64_t ldxz, void* cs, const float* cw, const float* cb,
                               void* u, int64_t ldu, int batch, int Ek, int K, float* zero0, int64_t nzero0,
                               float* zero1, int64_t nzero1, float* xacc, cudaStream_t s) {
  const int n = batch * Ek;
  if (n <= 0) return cudaSuccess;
  if ((nzero0 | nzero1) & 3) return cudaErrorInvalidValue;
  float4* z0 = reinterpret_cast<float4*>(zero0);
  float4* z1 = reinterpret_cast<float4*>(zero1);
  if (bf16)
    { cudaError_t e_ = launch(conv_decode_kernel<__nv_bfloat16, true>, (n + 255) / 256, 256, 0, s, 
        reinterpret_cast<const __nv_bfloat16*>(xz), ldxz, reinterpret_cast<__nv_bfloat16*>(cs), cw, cb,
        reinterpret_cast<__nv_bfloat16*>(u), ldu, batch, Ek, K, z0, nzero0 / 4, z1, nzero1 / 4, xacc); if (e_ != cudaSuccess) return e_; }
  else
    { cudaError_t e_ = launch(conv_decode_kernel<float, false>, (n + 255) / 256, 256, 0, s, 
        reinterpret_cast<const float*>(xz), ldxz, reinterpret_cast<float*>(cs), cw, cb, reinterpret_cast<float*>(u),
        ldu, batch, Ek, K, z0, nzero0 / 4, z1, nzero1 / 4, xacc); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

cudaError_t launch_unpack(int bf16, Peers src, int nsrc, int64_t off, int M, int hloc, int R, int N, int rmsnorm,
                          float eps, void* dlow, float* BC, cudaStream_t s) {
  const int64_t warps = (int64_t)M * hloc;
  if (warps <= 0) return cudaSuccess;
  if (R + 2 * N > kMaxP) return cudaErrorInvalidValue;
  const int blocks = (int)((warps * 32 + 255) / 256);
  if (bf16)
    { cudaError_t e_ = launch(unpack_kernel<__nv_bfloat16>, blocks, 256, 0, s, src, nsrc, off, M, hloc, R, N, rmsnorm, eps,
                                                        reinterpret_cast<__nv_bfloat16*>(dlow), BC); if (e_ != cudaSuccess) return e_; }
  else
    { cudaError_t e_ = launch(unpack_kernel<float>, blocks, 256, 0, s, src, nsrc, off, M, hloc, R, N, rmsnorm, eps,
                                                reinterpret_cast<float*>(dlow), BC); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

template <typename T, int N, bool F>
static cudaError_t scan_t(const void* u, int64_t ldu, const void* dl, int64_t ldd, const void* z, int64_t ldz,
                          const float* BC, int64_t ldbc, const float* a_log, const float* d_skip, float* h,
                          int64_t hbs, void* g, int64_t ldg, int batch, int L, int nch, cudaStream_t s) {
  dim3 grid((nch + SC_THREADS - 1) / SC_THREADS, batch);
  constexpr int TT = sizeof(T) == 2 ? 16 : 8;
  const int64_t rows = (int64_t)batch * L;
  const int es = (int)sizeof(T);
  CUtensorMap mu, md, mz, mbc;
  if (rows > INT32_MAX || !encode_tmap_2d(&mu, u, rows, nch, ldu, es, SC_THREADS, TT) ||
      !encode_tmap_2d(&md, dl, rows, nch, ldd, es, SC_THREADS, TT) ||
      !encode_tmap_2d(&mz, z, rows, nch, ldz, es, SC_THREADS, TT) ||
      !encode_tmap_2d(&mbc, BC, rows, 2 * N, ldbc, 4, 2 * N, TT))
    return cudaErrorInvalidValue;
  { cudaError_t e_ = launch(scan_kernel<T, N, F>, grid, SC_THREADS, 0, s, mu, md, mz, mbc, a_log, d_skip, h, hbs,
                            reinterpret_cast<T*>(g), ldg, L, nch); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

cudaError_t launch_scan(int bf16, int fast, const void* u, int64_t ldu, const void* dl, int64_t ldd, const void* z,
                        int64_t ldz, const float* BC, int64_t ldbc, const float* a_log, const float* d_skip, float* h,
                        int64_t hbs, void* g, int64_t ldg, int batch, int L, int nch, int N, cudaStream_t s) {
  if (batch <= 0 || L <= 0 || nch <= 0) return cudaSuccess;
  if (N != 16 && N != 8) return cudaErrorInvalidValue;
  if (bf16) {
    if (N == 16) return fast ? scan_t<__nv_bfloat16, 16, true>(u, ldu, dl, ldd, z, ldz, BC, ldbc, a_log, d_skip, h, hbs, g, ldg, batch, L, nch, s)
                             : scan_t<__nv_bfloat16, 16, false>(u, ldu, dl, ldd, z, ldz, BC, ldbc, a_log, d_skip, h, hbs, g, ldg, batch, L, nch, s);
    return fast ? scan_t<__nv_bfloat16, 8, true>(u, ldu, dl, ldd, z, ldz, BC, ldbc, a_log, d_skip, h, hbs, g, ldg, batch, L, nch, s)
                : scan_t<__nv_bfloat16, 8, false>(u, ldu, dl, ldd, z, ldz, BC, ldbc, a_log, d_skip, h, hbs, g, ldg, batch, L, nch, s);
  }
  if (N == 16) return scan_t<float, 16, false>(u, ldu, dl, ldd, z, ldz, BC, ldbc, a_log, d_skip, h, hbs, g, ldg, batch, L, nch, s);
  return scan_t<float, 8, false>(u, ldu, dl, ldd, z, ldz, BC, ldbc, a_log, d_skip, h, hbs, g, ldg, batch, L, nch, s);
}

template <typename T, int N, bool F>
static cudaError_t dstep_t(const DStepArgs& a, Peers src, int nsrc, cudaStream_t s) {
  // wide dt_rank at large batch (Falcon-Mamba-7B: R = 256, batch 32): two batch rows per thread share
  // each W_dt load, so the 512-B rows are read batch / 8 times instead of batch / 4 (71.1 -> 69.2 us per
  // Falcon-Mamba-7B decode layer; four rows per thread 71.1)
  const int ipt = (a.R >= 256 && a.batch >= 4 * DS_BB * 2) ? 2 : 1;
  const size_t smem = dstep_smem(a.R, N, (int)sizeof(T), ipt);
  dim3 grid((a.Ek + DS_CH - 1) / DS_CH, (a.batch + DS_BB * ipt - 1) / (DS_BB * ipt));
  cudaError_t e_ = ipt == 1 ? launch(decode_step_kernel<T, N, F>, grid, DS_THREADS, smem, s, a, src, nsrc)
                            : launch(decode_step_kernel<T, N, F, 2>, grid, DS_THREADS, smem, s, a, src, nsrc);
  if (e_ != cudaSuccess) return e_;
  return cudaGetLastError();
}

cudaError_t launch_decode_step(int bf16, Peers src, int nsrc, int64_t src_off, int ldp, int rmsnorm, float eps,
                               const void* u, const void* z, int64_t ldz, const void* w_dt, const float* b_dt,
                               const float* a_log, const float* d_skip, float* h, void* g, int batch, int Ek, int R,
                               int N, int ch_per_head, float* zacc, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  if (!dstep_supported(bf16, R, N, ldp, ch_per_head) || nsrc < 1 || nsrc > kMaxTP) return cudaErrorInvalidValue;
  DStepArgs a{};
  a.src_off = src_off; a.ldp = ldp; a.rmsnorm = rmsnorm; a.eps = eps; a.u = u; a.z = z; a.ldz = ldz; a.w_dt = w_dt;
  a.b_dt = b_dt; a.a_log = a_log; a.d_skip = d_skip; a.h = h; a.g = g; a.batch = batch; a.Ek = Ek; a.R = R;
  a.cph = ch_per_head; a.zacc = zacc;
  if (bf16) return N == 16 ? dstep_t<__nv_bfloat16, 16, true>(a, src, nsrc, s) : dstep_t<__nv_bfloat16, 8, true>(a, src, nsrc, s);
  return N == 16 ? dstep_t<float, 16, false>(a, src, nsrc, s) : dstep_t<float, 8, false>(a, src, nsrc, s);
}

cudaError_t launch_rmsnorm(int bf16, const float* x, const float* w, float eps, void* y, int64_t M, int D,
                           cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (D % 4 || D > 16 * 128 * 4) return cudaErrorInvalidValue;
  if (bf16)
    { cudaError_t e_ = launch(rmsnorm_kernel<__nv_bfloat16>, (unsigned)M, 128, 0, s, x, w, eps, reinterpret_cast<__nv_bfloat16*>(y), M, D); if (e_ != cudaSuccess) return e_; }
  else
    { cudaError_t e_ = launch(rmsnorm_kernel<float>, (unsigned)M, 128, 0, s, x, w, eps, reinterpret_cast<float*>(y), M, D); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

cudaError_t launch_rowstats(const float* x, void* y, float* ss, int64_t M, int D, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (D % 4 || D > 16 * 128 * 4) return cudaErrorInvalidValue;
  cudaError_t e = launch(rowstats_kernel, (unsigned)M, 128, 0, s, x, reinterpret_cast<__nv_bfloat16*>(y), ss, M, D);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_ssq_finalize(const float* part, int nchunk, float* ss, int64_t M, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  cudaError_t e = launch(ssq_finalize_kernel, (unsigned)((M * 32 + 255) / 256), 256, 0, s, part, nchunk, ss, M);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_quantize(const float* x, int64_t n, int blk, int8_t* q, float* scale, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t nb = n / blk;
  const int blocks = (int)((nb * 32 + 255) / 256);
  switch (blk) {
    case 32: { cudaError_t e_ = launch(quantize_kernel<1>, blocks, 256, 0, s, x, nb, q, scale); if (e_ != cudaSuccess) return e_; } break;
    case 64: { cudaError_t e_ = launch(quantize_kernel<2>, blocks, 256, 0, s, x, nb, q, scale); if (e_ != cudaSuccess) return e_; } break;
    case 128: { cudaError_t e_ = launch(quantize_kernel<4>, blocks, 256, 0, s, x, nb, q, scale); if (e_ != cudaSuccess) return e_; } break;
    case 256: { cudaError_t e_ = launch(quantize_kernel<8>, blocks, 256, 0, s, x, nb, q, scale); if (e_ != cudaSuccess) return e_; } break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_qar_reduce(Peers src, int k, int64_t q_off, int64_t s_off, int64_t n, int blk, float* out,
                              int accumulate, cudaStream_t s, void* cpy, float* ssq, int D) {
  if (n <= 0) return cudaSuccess;
  if (cpy && (!ssq || D % 32 || n % D)) return cudaErrorInvalidValue;
  const int64_t n16 = n / 16;
  const RowOut ro{reinterpret_cast<__nv_bfloat16*>(cpy), ssq, D};
  { cudaError_t e_ = launch(qar_reduce_kernel, (int)((n16 + 255) / 256), 256, 0, s, src, k, q_off, s_off, n16, blk, out, accumulate, ro); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

// Two-shot int8 all-reduce (reading Q6).  Layout in every rank's buffer half at byte offset `off`:
// amax [n/blk] f32 | scale [n/blk] f32 | codes [n] i8 | sums [n/k] i16 (each 256-B aligned).
cudaError_t launch_qar_twoshot(Peers peers, int rank, int k, int64_t off, const float* x, int64_t n, int blk,
                               float* out, int accumulate, cudaStream_t s, void* cpy, float* ssq, int D) {
  if (cpy && (!ssq || D % 32 || n % D)) return cudaErrorInvalidValue;
  const RowOut ro{reinterpret_cast<__nv_bfloat16*>(cpy), ssq, D};
  if (n <= 0) return cudaSuccess;
  if (n % (16 * k) || n % blk || blk % 16) return cudaErrorInvalidValue;
  const int64_t nb = n / blk;
  auto a256 = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  const int64_t o_amax = off, o_scale = o_amax + a256(nb * 4), o_q = o_scale + a256(nb * 4), o_sum = o_q + a256(n);
  char* own = reinterpret_cast<char*>(peers.p[rank]);
  const int blocks = (int)((nb * 32 + 255) / 256);
  cudaError_t e_ = cudaSuccess;
#define QTS(VPL)                                                                                              \
  e_ = launch(amax_kernel<VPL>, blocks, 256, 0, s, x, nb, reinterpret_cast<float*>(own + o_amax));           \
  if (e_ != cudaSuccess) return e_;                                                                           \
  if ((e_ = launch_peer_barrier(peers, rank, k, s)) != cudaSuccess) return e_;                               \
  e_ = launch(quant_shared_kernel<VPL>, blocks, 256, 0, s, x, nb, peers, k, o_amax,                           \
              reinterpret_cast<int8_t*>(own + o_q), reinterpret_cast<float*>(own + o_scale));                 \
  if (e_ != cudaSuccess) return e_;
  switch (blk) {
    case 32: QTS(1) break;
    case 64: QTS(2) break;
    case 128: QTS(4) break;
    case 256: QTS(8) break;
    default: return cudaErrorInvalidValue;
  }
#undef QTS
  if ((e_ = launch_peer_barrier(peers, rank, k, s)) != cudaSuccess) return e_;
  const int64_t shard = n / k, s16 = shard / 16;
  e_ = launch(rs16_kernel, (int)((s16 + 255) / 256), 256, 0, s, peers, k, o_q, (int64_t)rank * shard, s16,
              reinterpret_cast<int16_t*>(own + o_sum));
  if (e_ != cudaSuccess) return e_;
  if ((e_ = launch_peer_barrier(peers, rank, k, s)) != cudaSuccess) return e_;
  const int64_t n16 = n / 16;
  e_ = launch(ag16_kernel, (int)((n16 + 255) / 256), 256, 0, s, peers, o_sum, shard, n16,
              reinterpret_cast<const float*>(own + o_scale), blk, out, accumulate, ro);
  if (e_ != cudaSuccess) return e_;
  return cudaGetLastError();
}

cudaError_t launch_w16_cast(int bf16, const float* x, int64_t n, void* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n % 8) return cudaErrorInvalidValue;
  const int64_t n8 = n / 8;
  const int blocks = (int)((n8 + 255) / 256);
  cudaError_t e_ = bf16 ? launch(w16_cast_kernel<__nv_bfloat16>, blocks, 256, 0, s, x, n8, reinterpret_cast<uint4*>(out))
                        : launch(w16_cast_kernel<__half>, blocks, 256, 0, s, x, n8, reinterpret_cast<uint4*>(out));
  if (e_ != cudaSuccess) return e_;
  return cudaGetLastError();
}

cudaError_t launch_w16_reduce(int bf16, Peers src, int k, int64_t off, int64_t n, float* out, int accumulate,
                              cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n % 8) return cudaErrorInvalidValue;
  const int64_t n8 = n / 8;
  const int blocks = (int)((n8 + 255) / 256);
  cudaError_t e_ = bf16 ? launch(w16_reduce_kernel<__nv_bfloat16>, blocks, 256, 0, s, src, k, off, n8, out, accumulate)
                        : launch(w16_reduce_kernel<__half>, blocks, 256, 0, s, src, k, off, n8, out, accumulate);
  if (e_ != cudaSuccess) return e_;
  return cudaGetLastError();
}

// Requantised two-shot (labelled variant).  Layout in every rank's half at byte offset `off`:
// codes [n] i8 | scales [n/blk] f32 | requantised shard codes [n/k] i8 | shard scales [n/k/blk] f32.
cudaError_t launch_qar_requant(Peers peers, int rank, int k, int64_t off, const float* x, int64_t n, int blk,
                               float* out, int accumulate, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n % ((int64_t)k * blk) || blk % 16) return cudaErrorInvalidValue;
  auto a256 = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  const int64_t nb = n / blk, shard = n / k;
  const int64_t o_q = off, o_s = o_q + a256(n), o_q2 = o_s + a256(nb * 4), o_s2 = o_q2 + a256(shard);
  char* own = reinterpret_cast<char*>(peers.p[rank]);
  cudaError_t e_ = launch_quantize(x, n, blk, reinterpret_cast<int8_t*>(own + o_q), reinterpret_cast<float*>(own + o_s), s);
  if (e_ != cudaSuccess) return e_;
  if ((e_ = launch_peer_barrier(peers, rank, k, s)) != cudaSuccess) return e_;
  const int64_t nbs = shard / blk;
  const int blocks = (int)((nbs * 32 + 255) / 256);
#define RQR(VPL) e_ = launch(rq_reduce_kernel<VPL>, blocks, 256, 0, s, peers, k, o_q, o_s, (int64_t)rank * shard, nbs, \
                             reinterpret_cast<int8_t*>(own + o_q2), reinterpret_cast<float*>(own + o_s2))
  switch (blk) {
    case 32: RQR(1); break;
    case 64: RQR(2); break;
    case 128: RQR(4); break;
    case 256: RQR(8); break;
    default: return cudaErrorInvalidValue;
  }
#undef RQR
  if (e_ != cudaSuccess) return e_;
  if ((e_ = launch_peer_barrier(peers, rank, k, s)) != cudaSuccess) return e_;
  const int64_t n16 = n / 16;
  e_ = launch(rq_gather_kernel, (int)((n16 + 255) / 256), 256, 0, s, peers, o_q2, o_s2, shard, n16, blk, out, accumulate);
  if (e_ != cudaSuccess) return e_;
  return cudaGetLastError();
}

cudaError_t launch_f32_reduce(Peers src, int k, int64_t off, int64_t n, float* out, int accumulate, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t n4 = n / 4;
  { cudaError_t e_ = launch(f32_reduce_kernel, (int)((n4 + 255) / 256), 256, 0, s, src, k, off, n4, out, accumulate); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

// Force-load every kernel of this translation unit (CUDA lazy loading would otherwise load
// a kernel at its first launch, which can wait on a spinning peer barrier of another
// virtual rank on the same device).
__global__ void gather_cols_kernel(Peers src, int k, int64_t off, int64_t M, int wv, uint4* __restrict__ out,
                                   int64_t ldo_v);
cudaError_t preload_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {
      (const void*)conv1d_silu_kernel<__nv_bfloat16, 2, true>, (const void*)conv1d_silu_kernel<__nv_bfloat16, 3, true>,
      (const void*)conv1d_silu_kernel<__nv_bfloat16, 4, true>, (const void*)conv1d_silu_kernel<float, 2, false>,
      (const void*)conv1d_silu_kernel<float, 3, false>, (const void*)conv1d_silu_kernel<float, 4, false>,
      (const void*)conv_state_update_kernel<__nv_bfloat16>, (const void*)conv_state_update_kernel<float>,
      (const void*)conv_decode_kernel<__nv_bfloat16, true>, (const void*)conv_decode_kernel<float, false>,
      (const void*)unpack_kernel<__nv_bfloat16>, (const void*)unpack_kernel<float>,
      (const void*)scan_kernel<__nv_bfloat16, 16, true>, (const void*)scan_kernel<__nv_bfloat16, 16, false>,
      (const void*)scan_kernel<__nv_bfloat16, 8, true>, (const void*)scan_kernel<__nv_bfloat16, 8, false>,
      (const void*)scan_kernel<float, 16, false>, (const void*)scan_kernel<float, 8, false>,
      (const void*)conv1d_silu_v3_kernel<2>, (const void*)conv1d_silu_v3_kernel<3>, (const void*)conv1d_silu_v3_kernel<4>,
      (const void*)decode_step_kernel<__nv_bfloat16, 16, true>, (const void*)decode_step_kernel<__nv_bfloat16, 8, true>,
      (const void*)decode_step_kernel<__nv_bfloat16, 16, true, 2>, (const void*)decode_step_kernel<__nv_bfloat16, 8, true, 2>,
      (const void*)decode_step_kernel<float, 16, false>, (const void*)decode_step_kernel<float, 8, false>,
      (const void*)rmsnorm_kernel<__nv_bfloat16>, (const void*)rmsnorm_kernel<float>,
      (const void*)quantize_kernel<1>, (const void*)quantize_kernel<2>, (const void*)quantize_kernel<4>,
      (const void*)quantize_kernel<8>, (const void*)qar_reduce_kernel, (const void*)f32_reduce_kernel,
      (const void*)w16_cast_kernel<__half>, (const void*)w16_reduce_kernel<__half>,
      (const void*)w16_cast_kernel<__nv_bfloat16>, (const void*)w16_reduce_kernel<__nv_bfloat16>, (const void*)amax_kernel<4>,
      (const void*)quant_shared_kernel<4>, (const void*)rs16_kernel, (const void*)ag16_kernel,
      (const void*)peer_barrier_kernel, (const void*)gather_cols_kernel, (const void*)rq_reduce_kernel<1>,
      (const void*)rq_reduce_kernel<2>, (const void*)rq_reduce_kernel<4>, (const void*)rq_reduce_kernel<8>,
      (const void*)rq_gather_kernel};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// AR#1 publish + barrier of the fused decode path at TP > 1: the fused in_proj accumulated this
// rank's x_proj partial into the state-local buffer xacc; copy it into the rank's symmetric
// buffer (where the peers read it), re-zero xacc for the next token, then the cross-rank barrier
// (the copies are ordered before the flag by bar.sync + the signalling threads' fence.sys).
__global__ void __launch_bounds__(256) publish_barrier_kernel(Peers bufs, int rank, int k, float* __restrict__ xacc,
                                                              int64_t n, int64_t dst_off) {
  pdl_trigger();
  pdl_wait();
  __shared__ uint32_t s_epoch;
  const int t = threadIdx.x;
  float* dst = reinterpret_cast<float*>(reinterpret_cast<char*>(bufs.p[rank]) + dst_off);
  for (int64_t i = t; i < n / 4; i += 256) {
    reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(xacc)[i];
    reinterpret_cast<float4*>(xacc)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int64_t i = 4 * (n / 4) + t; i < n; i += 256) {
    dst[i] = xacc[i];
    xacc[i] = 0.f;
  }
  uint32_t* own = reinterpret_cast<uint32_t*>(bufs.p[rank]);
  if (t == 0) s_epoch = atomicAdd(own + 32, 1u) + 1u;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  if (t < k) {
    fence_sys();
    st_release_sys(reinterpret_cast<uint32_t*>(bufs.p[t]) + rank, epoch);
  }
  __syncwarp();
  if (t < k) {
    const uint32_t* slot = own + t;
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(slot) - epoch) < 0) {
      if (globaltimer() - t0 > 20ull * 1000000000ull) {
        atomicExch(own + 16, 1u);
        break;
      }
    }
  }
  __syncwarp();
  fence_sys();
}

cudaError_t launch_publish_barrier(Peers bufs, int rank, int k, float* xacc, int64_t n, int64_t dst_off,
                                   cudaStream_t s) {
  if ((reinterpret_cast<uintptr_t>(xacc) & 15) || (dst_off & 15)) return cudaErrorInvalidValue;
  { cudaError_t e_ = launch(publish_barrier_kernel, 1, 256, 0, s, bufs, rank, k, xacc, n, dst_off); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

__global__ void gather_cols_kernel(Peers src, int k, int64_t off, int64_t M, int wv, uint4* __restrict__ out,
                                   int64_t ldo_v) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = M * k * wv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / ((int64_t)k * wv);
    const int rem = (int)(i % ((int64_t)k * wv));
    const int r = rem / wv, j = rem % wv;
    const uint4* sp = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(src.p[r]) + off);
    out[m * ldo_v + (int64_t)r * wv + j] = sp[m * wv + j];
  }
}

cudaError_t launch_gather_cols(Peers src, int k, int64_t off, int64_t M, int wbytes, void* out, int64_t ldo_bytes,
                               cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if ((wbytes | ldo_bytes | off) & 15) return cudaErrorInvalidValue;
  const int wv = wbytes / 16;
  const int64_t total = M * k * wv;
  const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  cudaError_t e_ = launch(gather_cols_kernel, blocks, 256, 0, s, src, k, off, M, wv, reinterpret_cast<uint4*>(out),
                          ldo_bytes / 16);
  if (e_ != cudaSuccess) return e_;
  return cudaGetLastError();
}

cudaError_t launch_peer_barrier(Peers bufs, int rank, int k, cudaStream_t s) {
  { cudaError_t e_ = launch(peer_barrier_kernel, 1, 32, 0, s, bufs, rank, k); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

}  // namespace ssm
