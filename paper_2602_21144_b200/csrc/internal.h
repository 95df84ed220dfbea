// internal.h — launchers shared between the kernels and the C-ABI layer (api.cu).
#pragma once
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
  // Any kind: a weight range the NEXT kernel streams.  When set, the GEMM launches on every SM and
  // the CTAs without a tile (the decode GEMMs have fewer tiles than SMs) issue L2 prefetches of
  // [pf, pf + pf_bytes) and exit: HBM time the tile CTAs leave idle fetches the successor's weights.
  const void* pf;
  int64_t pf_bytes;
  // Decode chain (TP = 1; ssm_mixer_decode_chained): the pre-norm RMSNorm of every layer folded
  // into the GEMMs around it.  in_proj: the B operand is bf16(residual) un-normalised and each
  // accumulator column n is scaled by rsqrt(ss[n] * ss_scale + ss_eps) (the per-row 1/rms factors
  // out of the contraction).  out_proj (split-K atomics into the residual): the last contributor
  // of an output tile (counter fin_cnt[m-tile], fin_need contributions, reset by the last) writes
  // bf16 of the final residual tile into fin_x [N][fin_ldx] (the next layer's B operand) and adds
  // the tile's per-row sums of squares into fin_ss.
  const float* ss;
  float ss_scale, ss_eps;
  int* fin_cnt;
  int fin_need;
  __nv_bfloat16* fin_x;
  int64_t fin_ldx;
  float* fin_ss;
  // EPI_DECODE_INPROJ (SURVEY.md §8 rows a1-a3 fused for one decode token).
  // Output rows m are in_proj features: m < Ek are x channels -> causal conv step over the cached
  // window cst + SiLU -> u (bf16 [N][Ek]) and the window shifted in place; Ek <= m < 2Ek are z
  // -> C[n * ldc + m] (bf16).  The CTA then contracts its 128 u channels with the matching
  // columns of W_x (mma.sync) and adds the partial x_proj [N][hl*P] into xacc (pre-zeroed).
  void* cst;                  // [N][K-1][Ek] bf16
  const float* cw;            // [Ek][K]
  const float* cb;            // [Ek]
  void* u;                    // [N][Ek] bf16
  const void* wx;             // [hl*P][Ek] bf16 (block-diagonal over local heads)
  float* xacc;                // [N][hl*P] fp32
  int Ek, K, P, hl, cph;
  // Stream-K fused decode in_proj (sk_acc != NULL): the (tile, k-block) space is cut evenly over
  // all SMs; a CTA holding part of a tile adds its partial accumulator into sk_acc
  // [m_tiles][N][128] fp32 (all-zero between calls) and bumps sk_cnt[m-tile]; the last of the
  // tile's contributors reads the sum back, re-zeroes it and runs the conv / x_proj epilogue.
  float* sk_acc;
  int* sk_cnt;
  // EPI_DECODE_INPROJ pre-norm (nres != NULL): the epilogue warps first write the B operand
  // itself, B[n][:] = bf16(nres[n][:] / sqrt(mean(nres[n][:]^2) + nres_eps)) (the layer's weightless
  // pre-norm RMSNorm, reading Q16; every CTA writes the same values), then release the B loads.
  const float* nres;
  float nres_eps;
  __nv_bfloat16* nx;
};

struct Peers {
  void* p[kMaxTP];
};

// Decode step run inside the decode out_proj GEMM as the producer of its B operand g: the idle
// epilogue warps of every CTA run decode-step units (dstep.cuh) while the weight stream starts,
// then a grid-wide barrier (all CTAs co-resident: grid <= SMs, 1 CTA/SM) releases the B loads.
struct DStepJob {
  int enabled;
  int bf16;
  int N;                          // d_state (16 or 8)
  const float* dbc;               // [batch][ldp] x_proj result (single source, no AR#1)
  unsigned long long* sync;       // grid-barrier counter (monotonic; one per layer state)
  // flattened DStepArgs fields
  int ldp, rmsnorm;
  float eps;
  const void* u;
  const void* z;
  int64_t ldz;
  const void* w_dt;
  const float* b_dt;
  const float* a_log;
  const float* d_skip;
  float* h;
  void* g;
  int batch, Ek, R, cph;
  // local != 0: channel-owned mode.  CTA i owns the k-block range (the d_inner channels) of split
  // i and runs every output m-tile for it; its epilogue warps first run the decode step for
  // exactly those channels (the step is channel-local, so no grid barrier), then the CTA's B
  // operand g is loaded.  h and g are written by their owner CTA only.  The dbc rows every CTA
  // reads are re-zeroed (for the next token's fused in_proj) by the last CTA to finish reading
  // them (counter rd_cnt, reset by that CTA).
  // local = Q >= 1 m-groups: CTA i = (k-split i / Q, m-group i % Q) runs the m-tiles q, q + Q, ...
  // of its split; the split's channels are divided over its Q CTAs for the decode step, which then
  // meet at a group barrier (grp_cnt[split], monotonic) before loading g of the whole split.
  int local;
  int* rd_cnt;
  int64_t ndbc;  // floats of dbc to re-zero (batch * ldp)
  unsigned long long* grp_cnt;
};

// ---- GEMM launchers (return cudaSuccess or the launch error) ----
// tcgen05/TMEM/TMA bf16 GEMM: A [M,K] row stride lda, B [N,K] row stride ldb (elements).
// ksplit > 1: data-parallel split-K; ksplit < 0: stream-K over all SMs (both need EPI_ATOMIC_F32).
// Requires lda*2 % 16 == 0, ldb*2 % 16 == 0, 16-B aligned bases.
// a_indep: A is a weight (independent of the predecessor kernel): under PDL the producer issues
// the first ring fill of A before griddepcontrol.wait.
// A_blocked: optional copy of A in the blocked layout (pack_blocked); TMA then reads contiguous
// 16 KB boxes (sequential weight streams for the decode GEMMs).
cudaError_t gemm_tc_bf16(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb, int M, int N,
                         int K, int ksplit, const Epilogue& epi, int num_sms, cudaStream_t s, bool a_indep = false,
                         const __nv_bfloat16* A_blocked = nullptr, const DStepJob* job = nullptr);
// experiment-only: copy the GEMM timeline buffer (16 u64 per CTA, SSM_GEMM_NOMMA bit 8)
cudaError_t gemm_trace_read(unsigned long long* host, int n);
size_t packed_blocked_bytes(int rows, int cols);
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
                               int N, int ch_per_head, float* zacc, cudaStream_t s, float* zero_ss = nullptr,
                               const void* pf = nullptr, int64_t pf_bytes = 0);
cudaError_t launch_rmsnorm(int bf16, const float* x, const float* w, float eps, void* y, int64_t M, int D,
                           cudaStream_t s);
// Decode chain start: x = bf16(residual) (un-normalised), ss[b] = sum_d residual[b][d]^2, and the
// out_proj finaliser counters zeroed.  residual [M][D] fp32.
cudaError_t launch_chain_begin(const float* x, __nv_bfloat16* y, float* ss, int* cnt, int ncnt, int64_t M, int D,
                               cudaStream_t s);
// int8 quantisation of n fp32 values in blocks of blk: q [n] int8, scale [n/blk] f32.
cudaError_t launch_quantize(const float* x, int64_t n, int blk, int8_t* q, float* scale, cudaStream_t s);
// out (+)= sum_r s_r q_r over k sources (fixed order 0..k-1).
cudaError_t launch_qar_reduce(Peers src, int k, int64_t q_off, int64_t s_off, int64_t n, int blk, float* out,
                              int accumulate, cudaStream_t s);
cudaError_t launch_f32_reduce(Peers src, int k, int64_t off, int64_t n, float* out, int accumulate, cudaStream_t s);
cudaError_t launch_f16_cast(const float* x, int64_t n, void* out, cudaStream_t s);
cudaError_t launch_qar_twoshot(Peers peers, int rank, int k, int64_t off, const float* x, int64_t n, int blk,
                               float* out, int accumulate, cudaStream_t s);
cudaError_t launch_f16_reduce(Peers src, int k, int64_t off, int64_t n, float* out, int accumulate, cudaStream_t s);
// Cross-rank barrier: advance this rank's device-side epoch counter, write it into slot[rank]
// of every peer's signal area, wait for all peers' slots in our own area to reach it
// (bounded; sets the error word on timeout).
cudaError_t launch_peer_barrier(Peers bufs, int rank, int k, cudaStream_t s);
// fused decode at TP > 1: copy the x_proj partial (state-local, n floats) into this rank's
// symmetric buffer at dst_off, re-zero it, then the cross-rank barrier
cudaError_t launch_publish_barrier(Peers bufs, int rank, int k, float* xacc, int64_t n, int64_t dst_off,
                                   cudaStream_t s);

// ---- persistent whole-stack decode (decode_mk.cu) ----
// One layer of the stack as the persistent decode kernel reads it (TP=1, bf16, one x_proj head).
struct MkLayer {
  const __nv_bfloat16* w_in_pk;   // pack_blocked(W_in [2Ek, D]): 128x64 tiles, row-tile-major
  const __nv_bfloat16* w_out_pk;  // pack_blocked(W_out [D, Ek])
  const __nv_bfloat16* w_x;       // [P, Ek]
  const __nv_bfloat16* w_dt;      // [Ek, R]
  const float* conv_w;            // [Ek, K]
  const float* conv_b;            // [Ek]
  const float* b_dt;              // [Ek]
  const float* a_log;             // [Ek, 16]
  const float* d_skip;            // [Ek]
  __nv_bfloat16* conv;            // cache: conv window [batch][K-1][Ek]
  float* h;                       // cache: h [batch][Ek][16]
  void* pad;
};
struct MkParams {
  const MkLayer* layers;
  int n_layers;
  float* resid;                   // [B][D] fp32, caller's residual (in/out)
  float* residT;                  // [D][BP] fp32, the residual stream while the kernel runs
  __nv_bfloat16* residB;          // bf16 copy of residT, K-major SW128 k-blocks [D/64][BP][64]: in_proj B
  float* xzT;                     // [2Ek][BP] fp32 in_proj accumulators (zero between layers)
  float* dbcT;                    // [2][P][BP] fp32 x_proj accumulators (double-buffered by epoch)
  float* ss;                      // [2][BP] sums of squares of the residual rows (by epoch)
  float* ssP;                     // [grid][BP] per-CTA sums of squares of the input residual
  __nv_bfloat16* gT;              // gated scan output, K-major SW128 k-blocks [Ek/64][BP][64]: out_proj B
  unsigned* cnt;                  // readiness counters (mk_cnt_layout), monotonic since bind
  unsigned* ep;                   // [grid] layers completed since bind, per CTA
  unsigned long long* bar;        // grid-barrier arrival counter (monotonic)
  unsigned* err;                  // device error word (barrier / pipeline timeout)
  int B, D, Ek, R, P, K;
  float eps;                      // pre-norm RMSNorm eps (weight 1, reading Q16)
  int rmsnorm;                    // Falcon dt/B/C RMSNorm (Q18)
  float rms_eps;
  int ring, nbr, ncmax, ngrp;     // weight-ring slots, B-ring slots, channels per CTA (max), groups
  unsigned long long* trace;      // optional (NULL = off): [grid][n_layers][32] globaltimer stamps
  int dbg;                        // experiment-only (SSM_MK_DBG)
};
// Counter block (u32 words, 32 B apart): cnt_x, cnt_fin, cnt_in[2Ek/128], rdy_g[Ek/64],
// cnt_out[D/128], rdy_res[D/128].
struct MkCnt {
  int x, fin, in, g, out, res, words;
};
inline __host__ __device__ MkCnt mk_cnt_layout(int D, int Ek) {
  MkCnt c{};
  int o = 0;
  c.x = o; o += 8;
  c.fin = o; o += 8;
  c.in = o; o += 8 * (2 * Ek / 128);
  c.g = o; o += 8 * (Ek / 64);
  c.out = o; o += 8 * (D / 128);
  c.res = o; o += 8 * (D / 128);
  c.words = o;
  return c;
}
size_t mk_smem_bytes(int BP, int P, int R, int ncmax, int ring, int nbr);
int mk_ring_slots(int BP, int P, int R, int ncmax, int nbr);
cudaError_t launch_decode_mk(const MkParams& p, int BP, int grid, cudaStream_t s);
cudaError_t preload_decode_mk();

// Load every kernel eagerly (called once per process from ssm_tp_init when a device exists).
cudaError_t preload_kernels();
cudaError_t preload_gemm_simt();
cudaError_t preload_gemm_tc();

}  // namespace ssm
