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
#include <cstdlib>
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
  int nomma;         // experiment knob: skip the MMAs (TMA pipeline only)
};
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (2 per TMEM lane group)

// Work decomposition.  Data-parallel mode: unit u = (k-split, m-tile, n-tile), CTAs stride
// over units.  Stream-K mode (streamk != 0): the linearised (tile, k-block) space is cut into
// gridDim.x equal contiguous ranges, one per CTA; a range may cover the tail of one tile and
// the head of the next, so partial tiles are combined by the atomic epilogue.
struct TileSched {
  int m_tiles, n_tiles, kb_total, kbs, ksplit, units, streamk;
  // iterate segments (mt, nt, kb0, kb1) of this CTA; returns false when done
  __device__ bool next(int& cursor, int& mt, int& nt, int& kb0, int& kb1) const {
    if (!streamk) {
      const int u = cursor;
      if (u >= units) return false;
      cursor += gridDim.x;
      nt = u % n_tiles;
      const int rest = u / n_tiles;
      mt = rest % m_tiles;
      const int ks = rest / m_tiles;
      kb0 = ks * kbs;
      kb1 = min(kb_total, kb0 + kbs);
      return true;
    }
    const long long W = (long long)m_tiles * n_tiles * kb_total;
    const long long end = W * (blockIdx.x + 1) / gridDim.x;
    long long pos = cursor < 0 ? W * blockIdx.x / gridDim.x : (long long)cursor;
    if (pos >= end) return false;
    const int tile = (int)(pos / kb_total);
    kb0 = (int)(pos % kb_total);
    kb1 = (int)min((long long)kb_total, kb0 + (end - pos));
    nt = tile % n_tiles;
    mt = tile / n_tiles;
    cursor = (int)(pos + (kb1 - kb0));
    return true;
  }
  __device__ int first() const { return streamk ? -1 : (int)blockIdx.x; }
};

// Epilogue for one warp's 32 x 32 chunk: lane = row m0 + lane, columns n0..n0+31, stored
// straight from registers (staging through shared memory would compete with the UMMA operand
// reads for smem bandwidth in the MMA-bound projections).
__device__ __forceinline__ void epi_chunk(const Epilogue& e, int m0, int n0, int M, int N, uint32_t (&r)[32]) {
  const int kind = e.kind;
  const int m = m0 + threadIdx.x % 32;
  if (m >= M) return;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (kind == EPI_SOFTPLUS_BF16 || kind == EPI_SOFTPLUS_F32) {
    float bb[32];
    if (e.trans) {
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
    if (kind == EPI_SOFTPLUS_BF16) {  // bf16 output: 2-MUFU softplus (error far below bf16 rounding)
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = v[j] + bb[j];
        const float sp = 0.6931471805599453f * __log2f(1.f + ex2_approx(x * 1.4426950408889634f));
        v[j] = x > 20.f ? x : sp;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = softplus(v[j] + bb[j]);
    }
  }
  if (e.trans) {
    // element (m, n) -> C[n * ldc + m]; lanes hold consecutive m -> coalesced per n
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      if (n >= N) continue;
      const int64_t idx = (int64_t)n * e.ldc + m;
      switch (kind) {
        case EPI_STORE_BF16:
        case EPI_SOFTPLUS_BF16: reinterpret_cast<__nv_bfloat16*>(e.C)[idx] = __float2bfloat16_rn(v[j]); break;
        case EPI_STORE_F32:
        case EPI_SOFTPLUS_F32: reinterpret_cast<float*>(e.C)[idx] = v[j]; break;
        case EPI_ADD_F32: reinterpret_cast<float*>(e.C)[idx] += v[j]; break;
        default: atomicAdd(reinterpret_cast<float*>(e.C) + idx, v[j]);
      }
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
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) C[j] += v[j];
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

__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int BN, int KBS, TileSched ts, Epilogue epi, const __nv_bfloat16* a_pf, int64_t lda, int K,
                   CtaRes cr, int a_blocked) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int STAGES = num_stages(BN, KBS, cr.ring);
  const int SB = stage_bytes(BN, KBS);
  const int BOFF = KBS * A_STAGE;  // B tiles follow the KBS A tiles (1024-B aligned)
  const int BSUB = BN * BK * 2;
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
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, cr.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // A is the weight operand (swap-AB decode): stream this CTA's whole A range into L2 as long
    // contiguous row segments (DRAM-friendly) while the predecessor kernel finishes
    if (a_pf) {
      int cur = ts.first(), mt, nt, kb0, kb1;
      while (ts.next(cur, mt, nt, kb0, kb1)) {
        const int c0 = kb0 * BK;
        const int c1 = min(K, kb1 * BK);
        if (c1 <= c0) continue;
        for (int r = mt * BM + lane; r < min(M, mt * BM + BM); r += 32)
          prefetch_l2(a_pf + (int64_t)r * lda + c0, (uint32_t)(c1 - c0) * 2);
      }
    }
    pdl_wait();
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t ph = 0;
      int cur = ts.first(), mt, nt, kb0, kb1;
      while (ts.next(cur, mt, nt, kb0, kb1)) {
        for (int kb = kb0; kb < kb1; kb += KBS) {
          const int nk = min(KBS, kb1 - kb);
          mbar_wait(&empty[stage], ph ^ 1);
          mbar_arrive_expect_tx(&full[stage], (uint32_t)nk * (BM + BN) * BK * 2);
          uint8_t* st = ring + stage * SB;
          if (a_blocked)  // A pre-tiled: block (mt, kb) is one contiguous 16 KB box
            for (int j = 0; j < nk; ++j)
              tma_load_3d(st + j * A_STAGE, &tmA, &full[stage], 0, 0, mt * ts.kb_total + kb + j);
          else
            for (int j = 0; j < nk; ++j) tma_load_2d(st + j * A_STAGE, &tmA, &full[stage], (kb + j) * BK, mt * BM);
          for (int j = 0; j < nk; ++j) tma_load_2d(st + BOFF + j * BSUB, &tmB, &full[stage], (kb + j) * BK, nt * BN);
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      const uint32_t idesc = umma_idesc_bf16(BM, BN);
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
          const uint32_t s0 = smem_u32(ring + stage * SB);
          for (int j = 0; j < nk; ++j) {
            const uint32_t a0 = s0 + j * A_STAGE;
            const uint32_t b0 = s0 + BOFF + j * BSUB;
            if (!cr.nomma) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                umma_bf16(d, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                          (kb > kb0 || j > 0 || k > 0) ? 1u : 0u);
              }
            }
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9; TMEM lane group = warp % 4, column half = (warp-2)/4
    pdl_wait();
    const int eg = warp & 3;
    const int half = (warp - 2) >> 2;
    int acc = 0;
    uint32_t acc_ph = 0;
    int cur = ts.first(), mt, nt, kb0, kb1;
    while (ts.next(cur, mt, nt, kb0, kb1)) {
      if (kb0 >= kb1) continue;
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const int m0 = mt * BM + eg * 32;
      const uint32_t tbase = tmem_base + ((uint32_t)(eg * 32) << 16) + (uint32_t)(acc * cr.acc_stride);
      for (int c = half; c < BN / 32; c += 2) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tbase + c * 32, r);
        tmem_ld_wait();
        epi_chunk(epi, m0, nt * BN + c * 32, M, N, r);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, cr.tmem_cols);
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
// contiguous 16 KB row-major tile; blocks ordered row-tile-major.  TMA views it as a 3D tensor
// {64, 128, n_blocks} so every box is one contiguous 16 KB read (sequential weight streams).
bool make_map_blocked(CUtensorMap* map, const void* ptr, int64_t n_blocks) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)BK, (cuuint64_t)BM, (cuuint64_t)n_blocks};
  cuuint64_t strides[2] = {(cuuint64_t)(BK * 2), (cuuint64_t)(BK * BM * 2)};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)BM, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

__global__ void pack_blocked_kernel(const __nv_bfloat16* __restrict__ w, int rows, int cols, int64_t ld,
                                    __nv_bfloat16* __restrict__ out, int kbt, int64_t n_vec) {
  // one thread per 16-B output vector (8 bf16); zero padding beyond rows / cols
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_vec; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = v * 8;
    const int64_t blk = e / (BM * BK);
    const int within = (int)(e % (BM * BK));
    const int r = (int)(blk / kbt) * BM + within / BK;
    const int k = (int)(blk % kbt) * BK + within % BK;
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

cudaError_t preload_gemm_tc() {
  cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)gemm_tc_kernel);
}

bool gemm_tc_supported(const void* A, int64_t lda, const void* B, int64_t ldb) {
  return ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0) &&
         ((lda * 2) % 16 == 0) && ((ldb * 2) % 16 == 0) && get_encode() != nullptr;
}

cudaError_t gemm_tc_bf16(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb, int M, int N,
                         int K, int ksplit, const Epilogue& epi, int num_sms, cudaStream_t s, bool prefetch_a,
                         const __nv_bfloat16* A_blocked) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int ksplit_in = ksplit;
  // BN: multiple of 32 in [32, 256] (UMMA needs N % 16 == 0; the epilogue drains TMEM in
  // 32-column chunks) covering N in as few tiles as possible
  int n_tiles = (N + BN_MAX - 1) / BN_MAX;
  int BN = (N + n_tiles - 1) / n_tiles;
  BN = (BN + 31) / 32 * 32;
  n_tiles = (N + BN - 1) / BN;
  TileSched ts;
  ts.m_tiles = (M + BM - 1) / BM;
  ts.n_tiles = n_tiles;
  ts.kb_total = (K + BK - 1) / BK;
  if (ksplit < 1) ksplit = 1;
  if (ksplit > ts.kb_total) ksplit = ts.kb_total;
  ts.kbs = (ts.kb_total + ksplit - 1) / ksplit;
  ts.ksplit = (ts.kb_total + ts.kbs - 1) / ts.kbs;
  ts.units = ts.m_tiles * ts.n_tiles * ts.ksplit;
  ts.streamk = 0;
  if (ksplit_in < 0) {  // stream-K over all SMs (atomic epilogue)
    ts.streamk = 1;
    ts.ksplit = 1;
    ts.kbs = ts.kb_total;
    ts.units = ts.m_tiles * ts.n_tiles;
  }
  if ((ts.ksplit > 1 || ts.streamk) && epi.kind != EPI_ATOMIC_F32) return cudaErrorInvalidValue;

  CUtensorMap ma, mb;
  if (A_blocked) {
    if (!make_map_blocked(&ma, A_blocked, (int64_t)ts.m_tiles * ts.kb_total)) return cudaErrorInvalidValue;
  } else if (!make_map(&ma, A, M, K, lda, BM)) {
    return cudaErrorInvalidValue;
  }
  if (!make_map(&mb, B, N, K, ldb, BN)) return cudaErrorInvalidValue;

  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  // k-blocks per stage: skinny-N (weight-streaming) GEMMs fetch longer contiguous row segments
  int kbs = BN <= 64 ? 2 : 1;
  if (const char* env = getenv("SSM_GEMM_KBS")) kbs = atoi(env);
  if (kbs < 1) kbs = 1;
  CtaRes cr;
  cr.ring = RING_BYTES;
  cr.acc_stride = BN_MAX;
  cr.tmem_cols = 512;
  cr.nomma = 0;
  if (const char* env = getenv("SSM_GEMM_NOMMA")) cr.nomma = atoi(env);
  if (const char* env = getenv("SSM_GEMM_RING_KB")) {  // experiment: smaller CTA footprint
    cr.ring = atoi(env) * 1024;
    int cols = 32;
    while (cols < 2 * BN) cols *= 2;
    cr.tmem_cols = cols;
    cr.acc_stride = cols / 2;
  }
  while (kbs > 1 && num_stages(BN, kbs, cr.ring) < 2) --kbs;
  const int smem_bytes = 1024 + cr.ring + 512;
  int grid = ts.units < num_sms ? ts.units : num_sms;
  if (ts.streamk) {
    long long cap = num_sms;
    if (const char* env = getenv("SSM_GEMM_SK_CTAS")) cap = atoi(env);
    const long long W = (long long)ts.units * ts.kb_total;
    grid = (int)(W < cap ? W : cap);
  }
  { cudaError_t e_ = launch(gemm_tc_kernel, grid, kThreads, smem_bytes, s, ma, mb, M, N, BN, kbs, ts, epi,
                                      prefetch_a && !A_blocked && ((lda * 2) % 16 == 0) && (K % 8 == 0) ? A : nullptr,
                                      lda, K, cr, A_blocked ? 1 : 0); if (e_ != cudaSuccess) return e_; }
  return cudaGetLastError();
}

}  // namespace ssm
