// internal.h — launchers shared between the kernels and the C-ABI layer (api.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace ssm {

constexpr int kMaxTP = 8;
constexpr int kMaxState = 16;

// GEMM epilogue: C = A B^T (+ op).  Logical output element (m, n), m < M rows of A,
// n < N rows of B.  trans = 1 stores C[n * ldc + m] (swap-AB decode: A = weights).
enum EpiKind : int {
  EPI_STORE_BF16 = 0,     // C bf16 = acc
  EPI_STORE_F32 = 1,      // C f32 = acc
  EPI_SOFTPLUS_BF16 = 2,  // C bf16 = softplus(acc + bias[feature])
  EPI_SOFTPLUS_F32 = 3,   // C f32  = softplus(acc + bias[feature])
  EPI_ADD_F32 = 4,        // C f32 += acc            (read-modify-write; ksplit must be 1)
  EPI_ATOMIC_F32 = 5,     // C f32 += acc atomically (split-K; C pre-initialised)
  EPI_DECODE_INPROJ = 6,  // decode in_proj (swap-AB, bf16, N = batch <= 32), fused conv + x_proj; see below
  EPI_SPLIT_DBC = 8,      // x_proj at TP = 1 (no AR#1): column n = hd P + c of row m -> c < R: bf16 into
                          // dlow[(hd M + m) R + c], else fp32 into BC[(hd M + m) 2N + c - R] (the unpack
                          // layout; trans = 0, R % 32 == 0, P % 32 == 0, ldc = P, M = rows; fields dbc_*)
  EPI_QUANT_I8 = 7,       // int8 per-block quantisation of the accumulator (prefill out_proj at TP > 1, the
                          // one-shot AR#2 schedule): per qblk consecutive columns n of a row m, amax = max |acc|,
                          // s = fl32(amax / 127), code = clamp(rint(fl32(acc / s)), +-127) (0 if s == 0) ->
                          // C (int8 [M][ldc]), s -> qs[m * (N / qblk) + n / qblk]; trans = 0, N % qblk == 0
};

struct Epilogue {
  int kind;
  int trans;
  void* C;
  int64_t ldc;
  const float* bias;  // indexed by the output feature: n (trans=0) or m (trans=1)
  // Any kind: CTA 0 zero-fills zero[0, nzero) floats (16-B aligned) before its first tile -- a
  // buffer a LATER kernel accumulates into (saves a memset launch on the decode path).
  float* zero;
  int64_t nzero;
  // EPI_QUANT_I8: per-block scales and block size (32 | 64 | 128 | 256, dividing the tile width)
  float* qs;
  int qblk;
  // Optional row scale (kinds STORE_BF16 / STORE_F32 / ADD_F32 / ATOMIC_F32 / QUANT_I8): acc of the
  // logical row r (= m if trans = 0, n if trans = 1) is multiplied by 1 / sqrt(rss[r] * rss_inv +
  // rss_eps) before the store -- the gated RMSNorm's rstd applied after the out_proj contraction
  // (its weight is folded into the A operand by the scan; reading M3).
  const float* rss;
  float rss_inv, rss_eps;
  // Optional with EPI_ADD_F32 (trans = 0): the updated value is also stored as bf16 into cpy
  // ([M][ldc]) and each row's sum of squares over every 32-column chunk into ssq[m * ceil(N/32) + n/32]
  // (the next layer's pre-norm statistic without a separate pass; reading Q22).
  void* cpy;
  float* ssq;
  // EPI_DECODE_INPROJ (SURVEY.md §8 rows a1-a3 fused for one decode token).
  // Output rows m are in_proj features: m < Ek are x channels -> causal conv step over the cached
  // window cst + SiLU -> u (bf16 [N][Ek]) and the window shifted in place; Ek <= m < 2Ek are z
  // -> C[n * ldc + m] (bf16).  The CTA then contracts its 128 u channels with the matching
  // columns of W_x (mma.sync) and adds the partial x_proj [N][hl*P] into xacc (pre-zeroed).
  // EPI_SPLIT_DBC
  void* dbc_low;              // bf16 [hloc][M][R]
  float* dbc_bc;              // fp32 [hloc][M][2N]
  int dbc_R, dbc_P, dbc_M;
  void* cst;                  // [N][K-1][Ek] bf16
  const float* cw;            // [Ek][K]
  const float* cb;            // [Ek]
  void* u;                    // [N][Ek] bf16
  const void* wx;             // [hl*P][Ek] bf16 (block-diagonal over local heads)
  float* xacc;                // [N][hl*P] fp32
  int Ek, K, P, hl, cph;
};

struct Peers {
  void* p[kMaxTP];
};

// ---- GEMM launchers (return cudaSuccess or the launch error) ----
// tcgen05/TMEM/TMA bf16 GEMM: A [M,K] row stride lda, B [N,K] row stride ldb (elements).
// ksplit > 1: data-parallel split-K (needs EPI_ATOMIC_F32).
// Requires lda*2 % 16 == 0, ldb*2 % 16 == 0, 16-B aligned bases.
// a_indep: A is a weight (independent of the predecessor kernel): under PDL the producer issues
// the first ring fill of A before griddepcontrol.wait.
// A_blocked: optional copy of A in the blocked layout (pack_blocked); TMA then reads contiguous
// 16 KB boxes (sequential weight streams for the decode GEMMs).
cudaError_t gemm_tc_bf16(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb, int M, int N,
                         int K, int ksplit, const Epilogue& epi, int num_sms, cudaStream_t s, bool a_indep = false,
                         const __nv_bfloat16* A_blocked = nullptr);
size_t packed_blocked_bytes(int rows, int cols);
// 2D tensor map (no swizzle, zero fill out of bounds) of a row-major [rows x cols] matrix of bf16
// (elem_bytes 2) or fp32 (4) with row stride ld elements; box box_rows x box_cols.  False if the
// driver entry point is missing or the encode fails (pointer / stride not 16-B aligned).
bool encode_tmap_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int elem_bytes,
                    int box_cols, int box_rows);
cudaError_t pack_blocked(const __nv_bfloat16* w, int rows, int cols, int64_t ld, __nv_bfloat16* out, cudaStream_t s);
bool gemm_tc_supported(const void* A, int64_t lda, const void* B, int64_t ldb);
// SIMT GEMM, fp32 accumulation, T = float or bf16 inputs.
cudaError_t gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, int dtype_bf16, int M, int N, int K,
                      int ksplit, const Epilogue& epi, cudaStream_t s);

// ---- mixer kernels (T = bf16 if bf16 != 0 else float) ----
cudaError_t launch_conv1d_silu(int bf16, const void* xz, int64_t ldxz, const void* conv_state, const float* conv_w,
                               const float* conv_b, void* u, int64_t ldu, int batch, int L, int Ek, int K,
                               cudaStream_t s);
cudaError_t launch_conv_state_update(int bf16, const void* xz, int64_t ldxz, void* conv_state, int batch, int L,
                                     int Ek, int K, cudaStream_t s);
// Decode conv update; also zero-fills [zero0, zero0+nzero0) and [zero1, zero1+nzero1) floats
// (split-K accumulation targets of the next GEMMs; counts multiple of 4, 16-B aligned).
cudaError_t launch_conv_decode(int bf16, const void* xz, int64_t ldxz, void* conv_state, const float* conv_w,
                               const float* conv_b, void* u, int64_t ldu, int batch, int Ek, int K, float* zero0,
                               int64_t nzero0, float* zero1, int64_t nzero1, float* xacc, cudaStream_t s);
// Sum k_src fp32 partials [M, ldp] (fixed order), optional per-field RMSNorm, split into
// dt_low (T, [hloc][M][R]) and BC (f32, [hloc][M][2N]).
cudaError_t launch_unpack(int bf16, Peers src, int nsrc, int64_t src_off_bytes, int M, int hloc, int R, int N,
                          int rmsnorm, float eps, void* dlow, float* BC, cudaStream_t s);
cudaError_t launch_scan(int bf16, int fast, const void* u, int64_t ldu, const void* delta, int64_t ldd,
                        const void* z, int64_t ldz, const float* BC, int64_t ldbc, const float* a_log,
                        const float* d_skip, float* h, int64_t h_bstride, void* g, int64_t ldg, int batch, int L,
                        int nch, int N, cudaStream_t s);
// Decode step: sum of nsrc dbc partials [batch][ldp] at src_off (fixed order) (+RMSNorm),
// dt_proj + softplus, scan step, gate; h [batch][Ek][N] in place.
cudaError_t launch_decode_step(int bf16, Peers src, int nsrc, int64_t src_off, int ldp, int rmsnorm, float eps,
                               const void* u, const void* z, int64_t ldz, const void* w_dt, const float* b_dt,
                               const float* a_log, const float* d_skip, float* h, void* g, int batch, int Ek, int R,
                               int N, int ch_per_head, float* zacc, cudaStream_t s);
cudaError_t launch_rowstats(const float* x, void* y, float* ss, int64_t M, int D, cudaStream_t s);
cudaError_t launch_ssq_finalize(const float* part, int nchunk, float* ss, int64_t M, cudaStream_t s);
cudaError_t launch_rmsnorm(int bf16, const float* x, const float* w, float eps, void* y, int64_t M, int D,
                           cudaStream_t s);
// int8 quantisation of n fp32 values in blocks of blk: q [n] int8, scale [n/blk] f32.
cudaError_t launch_quantize(const float* x, int64_t n, int blk, int8_t* q, float* scale, cudaStream_t s);
// out (+)= sum_r s_r q_r over k sources (fixed order 0..k-1).  cpy != NULL: also the next layer's
// pre-norm inputs of the updated [n / D][D] rows: cpy = bf16(out) and per-32-column sums of squares -> ssq
// (launch_ssq_finalize forms the row statistic); D % 32 == 0.  Same for the two-shot schedule's all-gather.
cudaError_t launch_qar_reduce(Peers src, int k, int64_t q_off, int64_t s_off, int64_t n, int blk, float* out,
                              int accumulate, cudaStream_t s, void* cpy = nullptr, float* ssq = nullptr, int D = 0);
cudaError_t launch_f32_reduce(Peers src, int k, int64_t off, int64_t n, float* out, int accumulate, cudaStream_t s);
// Requantised two-shot int8 (labelled variant of reading Q6): quantise, barrier, shard owner sums and
// requantises, barrier, all-gather + dequantise; n % (k blk) == 0.
cudaError_t launch_qar_requant(Peers peers, int rank, int k, int64_t off, const float* x, int64_t n, int blk,
                               float* out, int accumulate, cudaStream_t s);
// 16-bit wire: fp16 (bf16 == 0) or bf16 RNE cast of n fp32 values (n % 8 == 0), and the fixed-order
// fp32 sum of the k ranks' 16-bit arrays.
cudaError_t launch_w16_cast(int bf16, const float* x, int64_t n, void* out, cudaStream_t s);
cudaError_t launch_w16_reduce(int bf16, Peers src, int k, int64_t off, int64_t n, float* out, int accumulate,
                              cudaStream_t s);
cudaError_t launch_qar_twoshot(Peers peers, int rank, int k, int64_t off, const float* x, int64_t n, int blk,
                               float* out, int accumulate, cudaStream_t s, void* cpy = nullptr, float* ssq = nullptr,
                               int D = 0);
// All-gather of column slices (naive TP arm): out[m][r * wbytes + j] = src_r[off + m * wbytes + j] for
// every rank r < k, bytes j < wbytes (multiple of 16); out row stride ldo_bytes.
cudaError_t launch_gather_cols(Peers src, int k, int64_t off, int64_t M, int wbytes, void* out, int64_t ldo_bytes,
                               cudaStream_t s);
// Cross-rank barrier: advance this rank's device-side epoch counter, write it into slot[rank]
// of every peer's signal area, wait for all peers' slots in our own area to reach it
// (bounded; sets the error word on timeout).
cudaError_t launch_peer_barrier(Peers bufs, int rank, int k, cudaStream_t s);
// fused decode at TP > 1: copy the x_proj partial (state-local, n floats) into this rank's
// symmetric buffer at dst_off, re-zero it, then the cross-rank barrier
cudaError_t launch_publish_barrier(Peers bufs, int rank, int k, float* xacc, int64_t n, int64_t dst_off,
                                   cudaStream_t s);

// ---- Zamba shared transformer block (attn.cu) ----
// mode 0: y = RMSNorm(concat(a, b)) * w over 2D columns; mode 1: y = RMSNorm(a + b) * w over D (b may
// be NULL); w may be NULL (ones); y bf16.
cudaError_t launch_rmsnorm2(const float* a, const float* b, int mode, const float* w, float eps, __nv_bfloat16* y,
                            int64_t M, int D, cudaStream_t s);
// K, V rows of qkv [batch*L][3 Hk d] -> cache [batch][Tmax][Hk][d] at the device-side length *len
// (err = 1 and nothing written on overflow); kv_advance: *len = min(*len + L, Tmax)
cudaError_t launch_kv_append(const __nv_bfloat16* qkv, const int* len, int batch, int L, int Hk, int d, int Tmax,
                             __nv_bfloat16* K, __nv_bfloat16* V, int* err, cudaStream_t s);
cudaError_t launch_kv_advance(int* len, int L, int Tmax, cudaStream_t s);
// causal attention of this call's queries (qkv) over the cache holding *len rows (this call's
// included); out [batch*L][Hk d] bf16; d in {32, 64, 128, 464}
cudaError_t launch_attn(const __nv_bfloat16* qkv, const int* len, const __nv_bfloat16* K, const __nv_bfloat16* V,
                        int batch, int L, int Hk, int d, int Tmax, float scale, __nv_bfloat16* out, cudaStream_t s);
// decode (L = 1) attention: split over the cached keys (flash decoding) + combine; part: workspace
// of attn_dec_part_floats floats
int attn_dec_splits(int batch, int Hk, int Tmax);
size_t attn_dec_part_floats(int batch, int Hk, int d, int Tmax);
cudaError_t launch_attn_decode(const __nv_bfloat16* qkv, const int* len, const __nv_bfloat16* K, const __nv_bfloat16* V,
                               int batch, int Hk, int d, int Tmax, float scale, float* part, __nv_bfloat16* out,
                               cudaStream_t s);
cudaError_t launch_gelu_mul(const __nv_bfloat16* gu, int64_t M, int I, __nv_bfloat16* m, cudaStream_t s);
cudaError_t launch_cast_bf16(const float* x, int64_t n, __nv_bfloat16* y, cudaStream_t s);
cudaError_t preload_attn();

// ---- Mamba-2 (SSD) mixer (ssd.cu) ----
cudaError_t launch_m2_scan(const __nv_bfloat16* proj, int64_t ldp, int dt_col, const __nv_bfloat16* u, int64_t ldu,
                           int b_col, int c_col, int heads_per_group, const float* dt_bias, const float* a_log,
                           const float* d_skip, const float* norm_w, float* hstate, __nv_bfloat16* o, int64_t ldo,
                           float* ss, int batch, int L, int Hk, int P, int N, cudaStream_t s);
cudaError_t preload_ssd();


// ---- persistent whole-stack decode at TP = 1 (decode_stack.cu) ----
struct DsLayer {            // one layer's device pointers (array in the plan's device buffer)
  const uint8_t* wa;        // in_proj units: 2E/8 units (x group i = unit 2i, z group i = unit 2i+1) x 16D B
  const uint8_t* wc;        // out_proj units: 4 quarters x D/8 row groups x 4E B (quarter-major)
  const uint32_t* wxf;      // x_proj B fragments [E/8][P/8][32] u32
  const uint8_t* wdt;       // dt_proj B fragments [E/8][R/16][32] x 8 B
  const float* conv_w;      // [E][K]
  const float* conv_b;      // [E]
  const float* b_dt;        // [E]
  const float* a_log;       // [E][16]
  const float* d_skip;      // [E]
  __nv_bfloat16* cst;       // conv window [B][K-1][E]
  float* h;                 // [B][E][16]
};

struct DsGeom {
  bool ok;
  int nch_max, ring_bytes, off_sb, off_red, off_pb, off_ut, off_misc, smem;
  size_t scratch_bytes;
};
DsGeom ds_geometry(int B, int D, int E, int R, int P, int K, int num_ctas);
size_t ds_packed_layer_bytes(int D, int E, int R, int P);
cudaError_t ds_pack_layer(const __nv_bfloat16* w_in, const __nv_bfloat16* w_out, const __nv_bfloat16* w_x,
                          const __nv_bfloat16* w_dt, int D, int E, int R, int P, uint8_t* dst, cudaStream_t s);
cudaError_t ds_fill_layer(DsLayer* host_entry, const uint8_t* packed, int D, int E, int R, int P,
                          const float* conv_w, const float* conv_b, const float* b_dt, const float* a_log,
                          const float* d_skip, void* cst, float* h);
cudaError_t ds_launch(const DsLayer* layers_dev, int L, int B, int D, int E, int R, int P, int K, float eps,
                      int bcdt_rmsnorm, float rms_eps, float* r, uint8_t* scratch, const DsGeom& g, int num_ctas,
                      cudaStream_t s, unsigned long long* trace = nullptr);
cudaError_t preload_decode_stack();
int ds_max_active(int smem);

// Load every kernel eagerly (called once per process from ssm_tp_init when a device exists).
cudaError_t preload_kernels();
cudaError_t preload_gemm_simt();
cudaError_t preload_gemm_tc();

}  // namespace ssm
