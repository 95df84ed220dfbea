// gemm_simt.cu — SIMT GEMM with fp32 accumulation for the fp32 mode (true fp32, no
// TF32: tcgen05 kind::tf32 keeps 10 mantissa bits and cannot hold the 1e-5 tolerance,
// SURVEY.md H6/Q20) and for shapes the TMA path cannot describe (row strides that are
// not multiples of 16 bytes).  Same epilogue contract as the tcgen05 GEMM.
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace ssm {
namespace {
constexpr int TM = 64, TN = 64, TK = 16;

__device__ __forceinline__ void epi_one(const Epilogue& e, int m, int n, float v) {
  if (e.kind == EPI_SOFTPLUS_BF16 || e.kind == EPI_SOFTPLUS_F32) v = softplus(v + e.bias[e.trans ? m : n]);
  if (e.rss) v *= rsqrtf(e.rss[e.trans ? n : m] * e.rss_inv + e.rss_eps);
  const int64_t idx = e.trans ? (int64_t)n * e.ldc + m : (int64_t)m * e.ldc + n;
  switch (e.kind) {
    case EPI_STORE_BF16:
    case EPI_SOFTPLUS_BF16:
      reinterpret_cast<__nv_bfloat16*>(e.C)[idx] = __float2bfloat16_rn(v);
      break;
    case EPI_STORE_F32:
    case EPI_SOFTPLUS_F32:
      reinterpret_cast<float*>(e.C)[idx] = v;
      break;
    case EPI_ADD_F32:
      reinterpret_cast<float*>(e.C)[idx] += v;
      break;
    default:
      atomicAdd(reinterpret_cast<float*>(e.C) + idx, v);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                                        int64_t ldb, int M, int N, int K, int kper, Epilogue epi) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sA[TK][TM + 4];
  __shared__ float sB[TK][TN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int kbeg = blockIdx.z * kper;
  const int kend = min(K, kbeg + kper);
  float acc[4][4] = {};
  for (int k0 = kbeg; k0 < kend; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      int r = i / TK, c = i % TK;
      int m = m0 + r, k = k0 + c;
      sA[c][r] = (m < M && k < kend) ? io<T>::ld(A + (int64_t)m * lda + k) : 0.f;
      int n = n0 + r;
      sB[c][r] = (n < N && k < kend) ? io<T>::ld(B + (int64_t)n * ldb + k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = sA[kk][ty * 4 + i];
        b[i] = sB[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) epi_one(epi, m, n, acc[i][j]);
    }
}
}  // namespace

cudaError_t preload_gemm_simt() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, (const void*)gemm_simt_kernel<float>);
  if (e != cudaSuccess) return e;
  return cudaFuncGetAttributes(&a, (const void*)gemm_simt_kernel<__nv_bfloat16>);
}

cudaError_t gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, int dtype_bf16, int M, int N, int K,
                      int ksplit, const Epilogue& epi, cudaStream_t s) {
  if (epi.kind == EPI_DECODE_INPROJ) return cudaErrorInvalidValue;  // tcgen05 path only
  if (epi.zero && epi.nzero > 0) {
    cudaError_t e = cudaMemsetAsync(epi.zero, 0, (size_t)epi.nzero * 4, s);
    if (e != cudaSuccess) return e;
  }
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (ksplit < 1) ksplit = 1;
  int kper = (K + ksplit - 1) / ksplit;
  kper = (kper + TK - 1) / TK * TK;
  if (kper <= 0) kper = TK;
  int nz = (K + kper - 1) / kper;
  if (nz < 1) nz = 1;
  if (nz > 1 && epi.kind != EPI_ATOMIC_F32) return cudaErrorInvalidValue;
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM, nz);
  if (dtype_bf16)
    { cudaError_t e_ = launch(gemm_simt_kernel<__nv_bfloat16>, grid, 256, 0, s, reinterpret_cast<const __nv_bfloat16*>(A), lda,
                                                         reinterpret_cast<const __nv_bfloat16*>(B), ldb, M, N, K,
                                                         kper, epi); if (e_ != cudaSuccess) return e_; }
  else
    { cudaError_t e_ = launch(gemm_simt_kernel<float>, grid, 256, 0, s, reinterpret_cast<const float*>(A), lda,
                                                 reinterpret_cast<const float*>(B), ldb, M, N, K, kper, epi); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

}  // namespace ssm
