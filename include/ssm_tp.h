/*
 * ssm_tp.h — C ABI of libssmtp.so: the tensor-parallel selective-SSM (Mamba)
 * mixer forward of arXiv 2602.21144 on B200 (sm_100a).
 *
 * The operation (§2.2 fig:mamba_mixer_block; §4.1-4.4):
 *   xz = x_in W_in,r^T               column-parallel in_proj, packed [x_r || z_r]
 *   u  = SiLU(causal_conv1d(x_r))    channel-separable, no communication
 *   dbc = AR#1( u W_x,r^T )          partial SSM-parameter projection + all-reduce
 *   dt_low, B, C = split(dbc)        column ranges [0,R) [R,R+N) [R+N,R+2N)
 *   delta = softplus(dt_low W_dt,r^T + b_dt,r)   "shard delta with channels"
 *   h_t = exp(delta A) h_{t-1} + delta B_t u_t ;  y_t = <C_t, h_t> + D u_t
 *   g  = y * SiLU(z)                 gate
 *   residual += AR#2( g W_out,r^T )  row-parallel out_proj, int8 quantised AR
 * with the SSM cache (conv window + h) carried from chunked prefill into decode
 * (§4.1).  Readings of points the paper leaves open are listed
 * in DESIGN.md §Readings.
 *
 * Conventions
 *  - Status: every function returns ssm_status_t (0 = OK).  The message of the
 *    last error on the calling thread is returned by ssm_last_error().
 *  - Ownership: the caller (PyTorch) allocates ALL device memory — weights,
 *    activations, state, workspace, symmetric communication buffers — and keeps
 *    it alive while handles that reference it exist.  The library never calls
 *    cudaMalloc; it owns only its host-side handles.
 *  - Streams: compute calls enqueue on the given stream and return.  Argument
 *    and shape errors are returned synchronously and nothing is enqueued.
 *    Device-side protocol failures (peer flag timeout) set an error word that
 *    ssm_tp_check() reports as SSM_ERR_PROTOCOL.
 *  - Collectives: with tp_size > 1, ssm_mixer_prefill/decode and
 *    ssm_qallreduce are collective: every rank calls them in the same order with
 *    the same (batch, seqlen, n, flags).  TP=1 performs no all-reduce and no
 *    quantisation (reading Q13).
 *  - Layouts: activations are token-major row-major [M x C], M = batch*seqlen,
 *    row m = b*seqlen + t, channels contiguous.  Weight matrices are nn.Linear
 *    [out, in] of the RANK-LOCAL shard (slicing the packed tensors per logical
 *    field is the caller's job — PAPER.md:336-345).  All pointers 16-B aligned.
 *  - dtype: SSM_BF16 = bf16 activations and weight matrices, fp32 accumulation,
 *    fp32 state, fp32 residual; SSM_FP32 = fp32 everywhere (true fp32 GEMMs,
 *    no TF32).  Per-channel vectors (conv_w, conv_b, b_dt, a_log, d_skip) are
 *    always fp32.
 *  - Threading: one ssm_tp_t per process/GPU; a handle is not thread-safe.
 *  - No fallback: there is no CPU path and no alternative backend.
 */
#ifndef SSM_TP_H
#define SSM_TP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SSM_OK = 0,
  SSM_ERR_ARG = 1,         /* null/misaligned pointer, bad flag, buffer too small              */
  SSM_ERR_DIM = 2,         /* shape mismatch                       */
  SSM_ERR_SHARD = 3,       /* d_inner % tp_size != 0, or heads not shardable */
  SSM_ERR_RANK = 4,        /* rank not in [0, tp_size)                            */
  SSM_ERR_CACHE = 5,       /* state does not belong to this handle / batch mismatch */
  SSM_ERR_PROTOCOL = 6,    /* collective timeout or order violation          */
  SSM_ERR_CUDA = 7,        /* CUDA runtime error                                               */
  SSM_ERR_UNSUPPORTED = 8  /* tp_size > 8, d_state > 16, qar_block does not divide d_model ... */
} ssm_status_t;

enum { SSM_BF16 = 0, SSM_FP32 = 1 };

/* flags for ssm_mixer_prefill / ssm_mixer_decode / ssm_qallreduce */
enum {
  SSM_AR2_INT8 = 0x1,      /* AR#2 = int8 per-block quantised all-reduce (default when tp>1)   */
  SSM_AR2_FP32 = 0x2,      /* AR#2 = exact fp32 one-shot all-reduce (unquantised arm)           */
  SSM_AR2_EXTERNAL = 0x4,  /* no AR#2: `residual` receives this rank's fp32 partial out_proj
                              (overwritten, not added) so the caller can all-reduce it itself
                              (the NCCL baseline arm)                                            */
  SSM_AR2_FP16 = 0x8,      /* AR#2 = the paper's FP32 -> FP16 wire: each rank
                              casts its fp32 partial to fp16 (IEEE RNE), exchanges it peer-to-peer,
                              and every rank forms sum_{r=0..k-1} fl32(h_r) in fp32, left to right
                              in rank order (reading Q21); the paper-literal ablation arm        */
  SSM_QAR_ACCUMULATE = 0x10, /* ssm_qallreduce: out += result instead of out = result           */
  SSM_QAR_FP16 = 0x20,      /* ssm_qallreduce: fp16 wire (as SSM_AR2_FP16) instead of int8 blocks;
                              n % 8 == 0                                                         */
  SSM_QAR_TWOSHOT = 0x40,   /* int8 schedule (reading Q6): shared per-block scales (amax max over
                              ranks), exact int16 reduce-scatter of the codes, all-gather of the
                              sums; wire (k-1)/k (n + 2n) B per rank instead of (k-1) n; bound
                              k max_r amax_r / 254.  ssm_qallreduce: selects it (n % (16 k) == 0);
                              mixer calls: forces it for SSM_AR2_INT8                           */
  SSM_QAR_ONESHOT = 0x80,   /* mixer calls: force the one-shot int8 schedule.  Default for
                              SSM_AR2_INT8: two-shot when tp_size >= 4 and the call has >= 64
                              tokens (prefill), one-shot otherwise (decode, k = 2)               */
  SSM_DECODE_UNFUSED = 0x100, /* ssm_mixer_decode: run the plain kernel chain (in_proj GEMM, conv
                              step, x_proj GEMM, decode step, out_proj) instead of the fused
                              in_proj (+conv step +x_proj epilogue); same arithmetic, used to
                              cross-check the fused kernel                                        */
  SSM_AR2_BF16 = 0x200,     /* AR#2 = custom bf16 wire (SURVEY.md §8(d) "custom bf16" arm, the
                              unquantised-16-bit baseline the int8 AR is compared with, PAPER.md
                              591-610): each rank casts its fp32 partial to bf16 (RNE), exchanges
                              it peer-to-peer, and every rank sums the k bf16 values in fp32 left
                              to right in rank order, added to the fp32 residual                 */
  SSM_QAR_BF16 = 0x400,     /* ssm_qallreduce: bf16 wire (as SSM_AR2_BF16); n % 8 == 0           */
  SSM_TP_NAIVE = 0x1000,    /* mixer calls, tp_size > 1, n_heads == 1: the paper's NAIVE sharding
                              baseline (§4.2 "the number of communication
                              collectives can grow to four per block"): W_in split uniformly
                              along its packed first extent (w_in_naive), so (i) the in_proj
                              output is all-gathered to rebuild the packed [x ; z] activation,
                              (ii) the conv output is all-gathered to rebuild the full-width
                              layout, then (iii) AR#1 on the x_proj partial and (iv) AR#2 at the
                              residual boundary, as in the channel-split design.  Same result;
                              four collectives per block instead of two.  Workspace:
                              ssm_workspace_bytes_flags(..., SSM_TP_NAIVE).  Ablation arm only. */
  SSM_QAR_REQUANT = 0x2000, /* int8 schedule, LABELLED VARIANT (never the default; reading Q6):
                              requantised two-shot -- per-rank scales as one-shot, the owner of
                              each 1/k shard sums the k ranks' dequantised codes in fp32 (rank
                              order) and requantises the sum with fresh per-block scales, then the
                              requantised shards are all-gathered.  Wire 2 (k-1)/k n (1 + 4/blk) B
                              per rank (k = 4: 1.55 n, 8: 1.80 n); bound 2 k max_r amax_r / 254.
                              ssm_qallreduce and SSM_AR2_INT8 mixer calls; n % (k qar_block) == 0 */
  SSM_QAR_FP32 = 0x4000     /* ssm_qallreduce: exact fp32 one-shot (no quantisation), fixed rank
                              order; n % 4 == 0                                                  */
};

enum { SSM_COMM_VIRTUAL = 0x1 }; /* ssm_comm_t.flags: all peer buffers live on THIS device
                                    (single-GPU virtual ranks, each driven on its own stream) */

typedef struct {
  int32_t d_model;       /* D                                                        */
  int32_t d_inner;       /* E = expand * D (global, unsharded)                        */
  int32_t d_state;       /* N <= 16                                                   */
  int32_t d_conv;        /* K, 2 <= K <= 8                                            */
  int32_t dt_rank;       /* R                                                        */
  int32_t n_heads;       /* x_proj groups H: 1 (Mamba, Falcon-Mamba) or 2 (Zamba);
                            channel d belongs to head d / (E/H) (reading Q17)           */
  int32_t dtype;         /* SSM_BF16 | SSM_FP32                                       */
  int32_t bcdt_rmsnorm;  /* 1: weightless RMSNorm on dt_low, B, C after AR#1 (Falcon-Mamba, Q18) */
  float rms_eps;         /* eps of that norm (1e-6)                                   */
  int32_t qar_block;     /* int8 block length along d_model (128; must divide D)      */
} ssm_config_t;

typedef struct {
  int32_t rank;          /* r in [0, tp_size)                                         */
  int32_t tp_size;       /* k in {1..8}                                               */
  void* const* peer_bufs;/* tp_size device pointers: the symmetric buffer of each rank,
                            mapped into this process (torch symmetric-memory rendezvous,
                            or same-device buffers with SSM_COMM_VIRTUAL).  peer_bufs[rank]
                            is this rank's own buffer.  May be NULL when tp_size == 1.  */
  size_t buf_bytes;      /* bytes of each symmetric buffer (>= ssm_comm_bytes())       */
  int32_t flags;         /* SSM_COMM_VIRTUAL or 0                                      */
} ssm_comm_t;

/* Rank-local weight shard of one mixer layer (E_k = d_inner / tp_size, P = R + 2N,
 * h_loc = max(1, n_heads / tp_size)).  Matrices in cfg.dtype, vectors fp32.       */
typedef struct {
  const void* w_in;      /* [2*E_k, D]  rows [0,E_k) = x of the owned channels,
                                        rows [E_k,2E_k) = z of the owned channels       */
  const float* conv_w;   /* [E_k, K]    tap K-1 multiplies the current token            */
  const float* conv_b;   /* [E_k]                                                       */
  const void* w_x;       /* [h_loc*P, E_k] block-diagonal over local heads              */
  const void* w_dt;      /* [E_k, R]                                                    */
  const float* b_dt;     /* [E_k]                                                       */
  const float* a_log;    /* [E_k, N]    A = -exp(a_log)                                 */
  const float* d_skip;   /* [E_k]                                                       */
  const void* w_out;     /* [D, E_k]                                                    */
  /* Optional (may be NULL): the same matrices pre-tiled by ssm_pack_weight.  When set, the
   * decode path streams them as contiguous 16 KB tiles (sequential HBM reads). bf16 only. */
  const void* w_in_pk;
  const void* w_x_pk;
  const void* w_out_pk;
  /* SSM_TP_NAIVE only: [2E/k, D] rows [r 2E/k, (r+1) 2E/k) of the PACKED W_in [x ; z] -- the
   * uniform split along the first extent that ignores the packed field boundary */
  const void* w_in_naive;
} ssm_layer_weights_t;

typedef struct ssm_tp_s* ssm_tp_t;
typedef struct ssm_state_s* ssm_state_t;

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* ssm_last_error(void);

/* Library version string. */
const char* ssm_version(void);

/* Validate cfg/comm and create a handle.  Errors: SSM_ERR_SHARD (d_inner % tp,
 * head split), SSM_ERR_RANK, SSM_ERR_UNSUPPORTED, SSM_ERR_ARG (buffer too small for
 * a zero-token call).  Allocates no device memory. */
ssm_status_t ssm_tp_init(const ssm_config_t* cfg, const ssm_comm_t* comm, ssm_tp_t* out);
ssm_status_t ssm_tp_destroy(ssm_tp_t tp);

/* Bytes of one rank's symmetric communication buffer for calls of up to
 * max_tokens (= batch*seqlen) tokens. */
ssm_status_t ssm_comm_bytes(const ssm_config_t* cfg, int32_t tp_size, int64_t max_tokens, size_t* bytes);

/* Bytes of the per-call workspace for (batch, seqlen); _flags: for calls with these flags
 * (SSM_TP_NAIVE needs the gathered full-width activations, M (3 d_inner) elements more). */
ssm_status_t ssm_workspace_bytes(ssm_tp_t tp, int32_t batch, int32_t seqlen, size_t* bytes);
ssm_status_t ssm_workspace_bytes_flags(ssm_tp_t tp, int32_t batch, int32_t seqlen, uint32_t flags, size_t* bytes);

/* SSM cache of one layer on this rank:
 *   conv window [batch][K-1][E_k] in cfg.dtype (raw x values, oldest first),
 *   h           [batch][E_k][N]   fp32.
 * ssm_state_bytes reports the two buffer sizes; ssm_state_alloc binds caller buffers of
 * at least those sizes and zero-fills them on `stream` (the prefill start state).  The h
 * buffer is h followed by library scratch of the fused decode path (x_proj accumulator,
 * grid-barrier counter) that must stay zero/monotonic between calls: never write it. */
ssm_status_t ssm_state_bytes(ssm_tp_t tp, int32_t batch, size_t* conv_bytes, size_t* h_bytes);
ssm_status_t ssm_state_alloc(ssm_tp_t tp, int32_t batch, void* conv_buf, size_t conv_bytes,
                             void* h_buf, size_t h_bytes, void* stream, ssm_state_t* out);
ssm_status_t ssm_state_reset(ssm_state_t st, void* stream);
ssm_status_t ssm_state_free(ssm_state_t st);

/* One mixer layer over a chunk of `seqlen` tokens for `batch` sequences, continuing
 * from the state (chunked prefill: call again with the next chunk).
 *   x_in     [batch*seqlen, D] cfg.dtype, replicated on all ranks (block input after the pre-norm)
 *   residual [batch*seqlen, D] fp32, replicated; residual += mixer(x_in)
 *            (with SSM_AR2_EXTERNAL: residual := this rank's partial out_proj)
 *   flags    SSM_AR2_INT8 | SSM_AR2_FP16 | SSM_AR2_FP32 | SSM_AR2_EXTERNAL (ignored when tp_size == 1)
 *   workspace >= ssm_workspace_bytes(batch, seqlen) bytes of device memory, 256-B aligned.
 * Errors: SSM_ERR_CACHE if st was allocated for another handle or batch;
 *         SSM_ERR_ARG if the symmetric buffer is too small for batch*seqlen tokens. */
ssm_status_t ssm_mixer_prefill(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st,
                               const void* x_in, float* residual, int32_t batch, int32_t seqlen,
                               uint32_t flags, void* workspace, size_t ws_bytes, void* stream);

/* Prefill of one pre-norm block with the norm folded around the projections (bf16; PAPER.md:151-174
 * with the pre-norm of reading Q16, rounding as reading Q22; at TP > 1 collective like ssm_mixer_prefill):
 *   residual += mixer(RMSNorm(residual))      (RMSNorm weight 1, eps norm_eps)
 * where x_in = bf16(residual) itself (NOT normalised) and ss_in[m] = sum_d residual[m][d]^2 (from
 * ssm_rowstats, or from the previous layer's call): the in_proj contracts bf16(r) and scales its row
 * m by 1 / sqrt(ss_in[m] / D + eps) in the epilogue, so no normalisation pass touches the residual.
 * If x_next / ss_next are given, the kernel that finishes the residual rows also writes
 * x_next = bf16(new residual) [batch*seqlen, D] and ss_next = its row sums of squares (fixed-order
 * reduction of per-32-column partials): the next layer's x_in / ss_in.  That kernel is the out_proj
 * epilogue that adds into the residual at TP = 1, and the int8 AR#2's dequantise-accumulate (one-shot
 * reduce or two-shot all-gather, §4.4) at TP > 1, so at no TP does a normalisation
 * pass touch the residual.  x_next may alias x_in (the in_proj has consumed it by then); ss_next must
 * not alias ss_in.  x_in, x_next and residual 16-B aligned, ss_in / ss_next 4-B aligned.
 * Errors: as ssm_mixer_prefill; SSM_ERR_UNSUPPORTED for fp32 handles, SSM_TP_NAIVE, strides the
 * tcgen05 GEMM cannot describe, and at tp_size > 1 an AR#2 other than int8 one- / two-shot or
 * d_model % 32 != 0 (use ssm_rmsnorm + ssm_mixer_prefill there). */
ssm_status_t ssm_mixer_prefill_normed(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st, const void* x_in,
                                      const float* ss_in, float norm_eps, float* residual, void* x_next,
                                      float* ss_next, int32_t batch, int32_t seqlen, uint32_t flags, void* workspace,
                                      size_t ws_bytes, void* stream);

/* x_out[m] = bf16(residual[m]) and ss_out[m] = sum_d residual[m][d]^2 for M rows of D = d_model (the first
 * layer's inputs of ssm_mixer_prefill_normed).  bf16 handles; 16-B aligned residual and x_out. */
ssm_status_t ssm_rowstats(ssm_tp_t tp, const float* residual, void* x_out, float* ss_out, int64_t M, void* stream);

/* One decode step (seqlen = 1) reading and updating the state in place.
 * Same arguments as prefill with seqlen = 1.  Graph-capturable. */
ssm_status_t ssm_mixer_decode(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st,
                              const void* x_in, float* residual, int32_t batch,
                              uint32_t flags, void* workspace, size_t ws_bytes, void* stream);

/* One pre-norm block of decode (PAPER.md:277-280 with the glue of reading Q16):
 *   residual += mixer(RMSNorm(residual))      (RMSNorm weight 1, eps norm_eps)
 * i.e. ssm_rmsnorm + ssm_mixer_decode with x_in in the workspace (the rmsnorm kernel, then the
 * decode kernels; graph-capturable).  residual [batch, D] fp32 in/out, 16-B aligned; workspace >=
 * ssm_workspace_bytes(batch, 1).  Errors as ssm_mixer_decode. */
ssm_status_t ssm_mixer_decode_block(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st, float* residual,
                                    int32_t batch, float norm_eps, uint32_t flags, void* workspace, size_t ws_bytes,
                                    void* stream);

/* ---- Persistent whole-stack decode at TP = 1 (§4.1) --------
 * ONE cooperative launch per token runs n_layers pre-norm decode blocks,
 *   for l in 0..n_layers-1:  residual += mixer_l(RMSNorm(residual))      (weight 1, eps norm_eps)
 * with the mixer of PAPER.md:151-174 (§2.2) at L = 1 from each layer's cached state: in_proj,
 * conv step + SiLU, x_proj, dt_proj + softplus, one scan step h = exp(dt A) h + dt B u (ZOH / Euler,
 * reading Q1), y = C h + D u, gate SiLU(z), out_proj.  Same result as n_layers calls of
 * ssm_mixer_decode_block up to rounding: the pre-norm's 1/rms is applied after the in_proj
 * contraction (in_proj(bf16(r)) * rstd instead of in_proj(bf16(r * rstd)); reading Q22)
 * and dt_low enters dt_proj in bf16.  Each SM streams its share of every layer's weights through a
 * shared-memory ring; grid barriers separate in_proj | scan step | out_proj.
 *   ssm_dstack_bytes:   bytes of the caller-owned device buffer for (n_layers, batch, ctas) (ctas = CTAs
 *                       of the launch, one per SM; 0 = all SMs).
 *   ssm_dstack_create:  binds `buf` (>= ssm_dstack_bytes, 256-B aligned): re-packs the layers' w_in,
 *                       w_out, w_x, w_dt into MMA-fragment order inside buf (the originals are not
 *                       referenced afterwards), keeps POINTERS to conv_w, conv_b, b_dt, a_log, d_skip and
 *                       to the states' conv window and h (updated in place by every decode: the same
 *                       caches ssm_mixer_prefill fills), zero-fills the scratch; synchronises `stream`.
 *                       layers / states: n_layers entries (host arrays).  The handle owns no device memory.
 *   ssm_dstack_decode:  residual [batch, D] fp32 (16-B aligned) in/out; graph-capturable (a cooperative
 *                       kernel node).  Every state is advanced by one token.
 * Errors: SSM_ERR_UNSUPPORTED unless tp_size 1, bf16, n_heads 1, d_state 16, batch <= 16, d_model % 128 == 0
 * and <= 2816, d_inner % 128 == 0 and <= 5632, dt_rank % 16 == 0; SSM_ERR_CACHE for a state of another
 * handle or batch; SSM_ERR_ARG for NULL pointers / a short or misaligned buffer / ctas > SMs. */
typedef struct ssm_dstack_s* ssm_dstack_t;
ssm_status_t ssm_dstack_bytes(ssm_tp_t tp, int32_t n_layers, int32_t batch, int32_t ctas, size_t* bytes);
ssm_status_t ssm_dstack_create(ssm_tp_t tp, int32_t n_layers, const ssm_layer_weights_t* layers,
                               const ssm_state_t* states, int32_t batch, float norm_eps, int32_t ctas, void* buf,
                               size_t buf_bytes, void* stream, ssm_dstack_t* out);
ssm_status_t ssm_dstack_decode(ssm_dstack_t ds, float* residual, void* stream);
ssm_status_t ssm_dstack_destroy(ssm_dstack_t ds);
/* Test/profiling only: subsequent ssm_dstack_decode calls write a timeline into `trace` (device,
 * ctas x n_layers x 32 u64 globaltimer stamps per CTA and layer: 0 layer start, 1 in_proj MMA done,
 * 2 in_proj epilogue done, 3 after barrier, 4 scan step done, 5 after barrier, 6 out_proj MMA done,
 * 7 out_proj epilogue done, 8 after barrier; 9 / 10 ns warp 0 waited for ring data in in_proj / out_proj;
 * 11-13 scan-step sub-phases; 16+i / 24+i in_proj epilogue: unit i started / its partials ready).
 * NULL switches it off. */
ssm_status_t ssm_dbg_dstack_trace(ssm_dstack_t ds, void* trace);

/* ---- Zamba's shared transformer block ------------------
 * Zamba runs one shared attention + MLP block before its 13 "hybrid" Mamba layers (the public
 * model definition, HF modeling_zamba.py: ZambaAttentionDecoderLayer + the hybrid layer's linear):
 *   x = RMSNorm_1(concat(h, h0)); q, k, v = x W_qkv^T (H heads of d = 2 D / H, no rotary)
 *   o = causal softmax(q k^T / sqrt(d / 2)) v over the KV cache; a = o W_o^T
 *   y = RMSNorm_2(a); m = (GELU(y W_g^T) * y W_u^T) W_d^T; t = m W_lin^T
 * and the hybrid layer's Mamba block then runs on RMSNorm(h + t) (ssm_rmsnorm_add) with residual h.
 * Tensor parallel (reading Z1): rank r owns heads [r H/k, (r+1) H/k) and MLP columns
 * [r I/k, (r+1) I/k) (column-parallel q/k/v and gate/up, row-parallel o and down, each followed by
 * an all-reduce; W_lin replicated).  bf16 handles only; d_model = the handle's d_model. */
typedef struct {
  int32_t n_heads;        /* H (global)                                                       */
  int32_t intermediate;   /* I (global)                                                       */
  float eps;              /* both RMSNorms (Zamba: 1e-5)                                      */
  int32_t max_seq;        /* KV cache capacity in tokens per sequence                         */
} ssm_attn_config_t;
typedef struct {          /* rank-local shards, bf16 matrices nn.Linear [out, in], fp32 vectors */
  const float* norm1;     /* [2D]                                                             */
  const void* w_qkv;      /* [3 (H/k) d, 2D]: rows q | k | v of the owned heads               */
  const void* w_o;        /* [D, (H/k) d]                                                     */
  const float* norm2;     /* [D]                                                              */
  const void* w_gu;       /* [2 I/k, D]: rows gate | up of the owned MLP columns              */
  const void* w_d;        /* [D, I/k]                                                         */
  const void* w_lin;      /* [D, D] (replicated)                                              */
} ssm_attn_weights_t;
typedef struct ssm_kv_s* ssm_kv_t;
/* KV cache of one shared-block application on this rank: caller-owned device buffer of
 * ssm_kv_bytes (256-B header with the device-side length, then K and V [batch][max_seq][H/k][d]
 * bf16); alloc binds and zero-fills it; reset empties it.  Calls append to it (prefill chunks,
 * decode tokens); the length lives in device memory, so a captured decode graph keeps appending. */
ssm_status_t ssm_kv_bytes(ssm_tp_t tp, const ssm_attn_config_t* acfg, int32_t batch, size_t* bytes);
ssm_status_t ssm_kv_alloc(ssm_tp_t tp, const ssm_attn_config_t* acfg, int32_t batch, void* buf, size_t bytes,
                          void* stream, ssm_kv_t* out);
ssm_status_t ssm_kv_reset(ssm_kv_t kv, void* stream);
ssm_status_t ssm_kv_free(ssm_kv_t kv);
ssm_status_t ssm_attn_workspace_bytes(ssm_tp_t tp, const ssm_attn_config_t* acfg, int32_t batch, int32_t seqlen,
                                      size_t* bytes);
/* t_out [batch*seqlen, D] fp32 := the block applied to h, h0 [batch*seqlen, D] fp32 (row = b L + t);
 * the call's K, V are appended to kv (SSM_ERR_PROTOCOL from ssm_tp_check if max_seq overflows).
 * flags: the two all-reduces at TP > 1: SSM_AR2_FP32 (exact, default when 0), SSM_AR2_INT8,
 * SSM_AR2_FP16, SSM_AR2_BF16.  Collective at TP > 1 (two all-reduces). */
ssm_status_t ssm_attn_block(ssm_tp_t tp, const ssm_attn_config_t* acfg, const ssm_attn_weights_t* w, ssm_kv_t kv,
                            const float* h, const float* h0, float* t_out, int32_t batch, int32_t seqlen,
                            uint32_t flags, void* workspace, size_t ws_bytes, void* stream);
/* x = RMSNorm(a + b) * weight (b may be NULL, weight may be NULL = ones), a, b fp32 [M, D] ->
 * x [M, D] in the handle's dtype: the hybrid layer's Mamba pre-norm of h + t. */
ssm_status_t ssm_rmsnorm_add(ssm_tp_t tp, const float* a, const float* b, const float* weight, float eps, void* x_out,
                             int64_t M, void* stream);

/* ---- Mamba-2 (SSD) mixer under the same TP design ----
 * Packed in_proj [z | x | B | C | dt], causal conv + SiLU over the x|B|C channels, the scalar-A-per-
 * head selective scan h <- exp(dt A) h + dt x B, y = C.h + D x (d_state N, head dim P = 64),
 * gated RMSNorm o = RMSNorm(y SiLU(z)) * w over d_inner (norm after the gate), out_proj.
 * Tensor parallel (reading M1): rank r owns heads [r H/k, (r+1) H/k) (z, x, dt rows of W_in, their
 * conv / dt_bias / A_log / D / norm entries, W_out columns); B and C (n_groups == 1) are replicated
 * on every rank (their W_in rows and conv taps too) -- no all-reduce before the scan; the gated
 * RMSNorm's per-token sum of squares is all-reduced (exact fp32, M floats), out_proj row-parallel
 * -> AR#2 into the residual (flags: SSM_AR2_INT8 one-shot, SSM_AR2_FP32, SSM_AR2_FP16, SSM_AR2_BF16).
 * The handle supplies d_model and the communicator; bf16 only.
 * Kernels: calls of >= 16 tokens scan in the chunked SSD (matmul) form (64-token chunks, d_state 64 or
 * 128), decode (seqlen 1) as one streaming step, other calls token by token; every scan writes
 * bf16(y SiLU(z) w) and the per-token sums of squares, and the out_proj applies 1/sqrt(ss/E + eps)
 * per row after the contraction (reading M3 in DESIGN.md). */
typedef struct {
  int32_t d_inner;        /* E (global)                                                       */
  int32_t d_state;        /* N: 16, 64 or 128                                                 */
  int32_t headdim;        /* P: 64                                                            */
  int32_t n_groups;       /* G: 1 (B/C replicated over the ranks)                             */
  int32_t d_conv;         /* K: 2..4                                                          */
  float eps;              /* gated RMSNorm                                                    */
} ssm_m2_config_t;
typedef struct {          /* rank-local: E_k = E/k, H_k = H/k, C_k = E_k + 2 G N             */
  const void* w_in;       /* [2 E_k + 2 G N + H_k, D] bf16: rows z_r | x_r | B | C | dt_r      */
  const float* conv_w;    /* [C_k, K]: x channels of the rank, then B, C                       */
  const float* conv_b;    /* [C_k]                                                           */
  const float* dt_bias;   /* [H_k]                                                           */
  const float* a_log;     /* [H_k]                                                           */
  const float* d_skip;    /* [H_k]                                                           */
  const float* norm_w;    /* [E_k]                                                           */
  const void* w_out;      /* [D, E_k] bf16                                                    */
} ssm_m2_weights_t;
/* cache of one layer on this rank: conv window [batch][K-1][C_k] bf16, h [batch][H_k][P][N] fp32 */
ssm_status_t ssm_m2_state_bytes(ssm_tp_t tp, const ssm_m2_config_t* cfg, int32_t batch, size_t* conv_bytes,
                                size_t* h_bytes);
ssm_status_t ssm_m2_workspace_bytes(ssm_tp_t tp, const ssm_m2_config_t* cfg, int32_t batch, int32_t seqlen,
                                    size_t* bytes);
/* residual [batch*seqlen, D] fp32 += mixer(x_in [batch*seqlen, D] bf16), row = b L + t; the cache
 * carries across calls (prefill chunks, then seqlen == 1 decode).  Caller-owned state buffers
 * (zero = empty cache).  Collective at TP > 1 (two all-reduces). */
ssm_status_t ssm_m2_mixer(ssm_tp_t tp, const ssm_m2_config_t* cfg, const ssm_m2_weights_t* w, void* conv_state,
                          float* h_state, const void* x_in, float* residual, int32_t batch, int32_t seqlen,
                          uint32_t flags, void* workspace, size_t ws_bytes, void* stream);

/* Quantised all-reduce of n fp32 values (n % qar_block == 0), rows of D = d_model:
 * every rank quantises its partial per block (s = amax/127, q = rint(o/s) clamped to
 * +-127), exchanges int8 codes + fp32 scales peer-to-peer, and forms
 * out = sum_{r=0..k-1} s_r q_r in fixed rank order in fp32 (bitwise identical on all
 * ranks).  out may alias partial.  tp_size == 1: out = partial (no quantisation).
 * n == 0 is a no-op (pointers may be NULL; with tp_size > 1 every rank must agree on it).
 * flags: SSM_QAR_ACCUMULATE, SSM_QAR_FP16, SSM_QAR_TWOSHOT (shared-scale two-shot schedule).
 * Error bound per element: sum_r s_r / 2 (int8 one-shot); k max_r amax_r / 254 (two-shot);
 * sum_r (|o_r| 2^-11 + 2^-25) + the fp32 additions (fp16 wire). */
ssm_status_t ssm_qallreduce(ssm_tp_t tp, const float* partial, float* out, size_t n,
                            uint32_t flags, void* stream);

/* Pre-norm glue (reading Q16): x[m,:] = residual[m,:] / sqrt(mean(residual[m,:]^2) + eps) * weight,
 * residual fp32 [M, D] -> x cfg.dtype [M, D]; weight fp32 [D] (may be NULL = ones). */
ssm_status_t ssm_rmsnorm(ssm_tp_t tp, const float* residual, const float* weight, float eps,
                         void* x_out, int64_t M, void* stream);

/* Pre-tiled copy of a bf16 weight matrix [rows, cols] (row-major, nn.Linear layout) for the
 * decode GEMMs: 128 x 64 tiles, each one contiguous 16 KB block, ordered row-tile-major and
 * zero-padded to whole tiles; inside a tile, row r's eight 16-B chunks are stored in the
 * SWIZZLE_128B order (chunk j at slot j ^ (r % 8)) so the tile is its own shared-memory image.
 * The layout is private to this library (consume it only through w_*_pk).  out must be 128-B
 * aligned and >= ssm_packed_weight_bytes bytes. */
ssm_status_t ssm_packed_weight_bytes(int32_t rows, int32_t cols, size_t* bytes);
ssm_status_t ssm_pack_weight(ssm_tp_t tp, const void* w, int32_t rows, int32_t cols, void* out, size_t out_bytes,
                             void* stream);

/* Synchronise the stream and report device-side protocol errors (SSM_ERR_PROTOCOL). */
ssm_status_t ssm_tp_check(ssm_tp_t tp, void* stream);

/* Collective counters: all-reduces issued by this handle, and the
 * bytes this rank wrote into its symmetric buffer for them. */
ssm_status_t ssm_tp_stats(ssm_tp_t tp, int64_t* allreduce_count, int64_t* bytes_sent);

/* Decode calls of this handle that ran the fused in_proj kernel (conv step and x_proj in the
 * GEMM epilogue; taken for bf16 when batch <= 32, P <= 320 and even, 2 <= K <= 4, 128 |
 * channels per head, and SSM_DECODE_UNFUSED is not set).  The other decode calls run the
 * unfused chain. */
ssm_status_t ssm_tp_fused_calls(ssm_tp_t tp, int64_t* calls);

/* Collective epoch of the handle: the number of collectives (all-reduces and barriers) this rank
 * has enqueued.  Collective e exchanges through half (e & 1) of the symmetric buffers, so two
 * consecutive collectives always use different halves.  A CUDA graph captured with the epoch at
 * parity p must be replayed with the epoch at parity p (its halves are fixed at capture);
 * ssm_tp_barrier realigns it. */
ssm_status_t ssm_tp_epoch(ssm_tp_t tp, uint32_t* epoch);
/* Cross-rank barrier with no payload (a collective: every rank calls it in the same order);
 * advances the epoch by one.  No-op (epoch unchanged) at tp_size == 1. */
ssm_status_t ssm_tp_barrier(ssm_tp_t tp, void* stream);

/* Kernel launches enqueued by this handle since creation (for bench.py gpu_launches). */
ssm_status_t ssm_tp_launch_count(ssm_tp_t tp, int64_t* launches);

/* Per-kernel timing probes (bench.py roofline): while enabled for `kernel`, the library records
 * a CUDA event pair on the launching stream around every launch of that kernel kind (outside
 * graph capture, except SSM_PROBE_IN_PROJ_DECODE), up to `capacity` launches.  Each kind has
 * its own slot; capacity 0 disables the kind and releases its events. */
enum { SSM_PROBE_IN_PROJ = 1, SSM_PROBE_CONV = 2, SSM_PROBE_X_PROJ = 3, SSM_PROBE_DT_PROJ = 4, SSM_PROBE_SCAN = 5,
       SSM_PROBE_OUT_PROJ = 6, SSM_PROBE_AR2 = 7, SSM_PROBE_DECODE_STEP = 8,
       SSM_PROBE_IN_PROJ_DECODE = 9 /* decode in_proj; recorded INSIDE graph capture too (event nodes:
                                       after replays, each pair holds its latest replay's times) */ };
ssm_status_t ssm_tp_probe(ssm_tp_t tp, int32_t kernel, int32_t capacity);
/* Synchronises the recorded events of `kernel` and writes up to `capacity` per-launch durations (ms). */
ssm_status_t ssm_tp_probe_read(ssm_tp_t tp, int32_t kernel, float* ms, int32_t capacity, int32_t* n);

/* ------------------------------------------------------------------ test-only */
/* C = A B^T with A [M,K], B [N,K] (cfg.dtype), C fp32 [M,N]; exercises the GEMM used
 * by the projections (tcgen05 for bf16 when K*2 % 16 == 0, SIMT otherwise). */
ssm_status_t ssm_dbg_gemm(ssm_tp_t tp, const void* A, const void* B, float* C,
                          int32_t M, int32_t N, int32_t K, int32_t swap_ab, int32_t ksplit, void* stream);
/* Selects the tcgen05 GEMM's CTA-pair variant (cta_group::2, M = 256 tiles over a 2-CTA cluster)
 * for every later call in the process: -1 = by shape (default: prefill GEMMs with M >= 4096,
 * N >= 128, K >= 1024, except the softplus dt_proj), 0 = never, 1 = whenever the call is eligible (non-transposed, no split-K,
 * M > 128).  Results are identical up to fp32 summation order inside the tensor core.  Returns
 * SSM_ERR_ARG for any other mode. */
ssm_status_t ssm_dbg_set_gemm_pair(int32_t mode);
/* Swap-AB decode GEMM C[M,N] = X[M,K] W[N,K]^T reading W through its packed copy Wpk. */
ssm_status_t ssm_dbg_gemm_packed(ssm_tp_t tp, const void* X, const void* W, const void* Wpk, float* C, int32_t M,
                                 int32_t N, int32_t K, int32_t ksplit, void* stream);
/* Same with explicit row strides (elements) of A and B. */
ssm_status_t ssm_dbg_gemm_ld(ssm_tp_t tp, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int32_t M,
                             int32_t N, int32_t K, int32_t swap_ab, int32_t ksplit, void* stream);
/* Selective scan + D skip + gate on prepared inputs (u, delta, z bf16/fp32 [batch*L, E_k],
 * z row stride ldz; BC fp32 [batch*L, 2N]); h [batch][E_k][N] fp32 in/out; g out. */
ssm_status_t ssm_dbg_scan(ssm_tp_t tp, const void* u, const void* delta, const void* z, int32_t ldz,
                          const float* BC, const float* a_log, const float* d_skip, float* h,
                          void* g, int32_t batch, int32_t seqlen, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSM_TP_H */
