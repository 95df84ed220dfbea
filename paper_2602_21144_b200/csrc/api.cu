// api.cu — C ABI of libssmtp (include/ssm_tp.h): validation, handles, workspace and
// symmetric-buffer layout, and the per-layer orchestration of the TP mixer
// (SURVEY.md §3 call stack (2)/(3); §4.1-4.4).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/ssm_tp.h"
#include "internal.h"
#include "dstep.cuh"

using namespace ssm;

namespace ssm {
thread_local bool t_launch_pdl = false;
int t_gemm_pair = -1;
}

namespace {

thread_local std::string g_err;

ssm_status_t fail(ssm_status_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                                   \
  do {                                                                                             \
    cudaError_t _e = (expr);                                                                       \
    if (_e != cudaSuccess) return fail(SSM_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// Programmatic dependent launch on the decode path: every kernel calls
// griddepcontrol.launch_dependents at entry and griddepcontrol.wait before touching memory a
// predecessor writes, so a successor's launch and prologue overlap the predecessor's tail
// (measured 45.3 -> 42.2 us per Mamba-2.8B decode layer with the fused in_proj).  Off across
// virtual ranks (see ssm_mixer_decode).
struct PdlScope {
  bool prev;
  explicit PdlScope(bool on) : prev(ssm::t_launch_pdl) { ssm::t_launch_pdl = on; }
  ~PdlScope() { ssm::t_launch_pdl = prev; }
};

constexpr size_t kSigBytes = 256;  // signal slots [0,32) B, error word at +64 B, epoch counter at +128 B

}  // namespace

struct ssm_tp_s {
  ssm_config_t cfg;
  int rank, k, flags;
  Peers peers;
  size_t buf_bytes;
  int Ek, P, hloc, cph;   // local channels, packed width, local heads, channels per local head
  int ar1_group;          // ranks summed by AR#1 (1 = no AR#1)
  int bf16, es;           // activation dtype flag and element size
  uint32_t epoch;
  int64_t ar_count, bytes_sent, launches;
  int num_sms;
  int64_t fused_calls;    // decode calls that took the fused in_proj (+conv step +x_proj) path
  // timing probes: one slot per kernel kind
  struct ProbeSlot {
    int cap = 0, n = 0;
    cudaEvent_t* ev = nullptr;  // 2 * cap events
  } probes[16];
};

struct ssm_state_s {
  ssm_tp_s* owner;
  int batch;
  void* conv;
  float* h;
};

struct ssm_kv_s {
  ssm_tp_s* owner;
  int batch, max_seq, hk, d;
  char* buf;  // header (int len @0, int err @4), K, V
};

namespace {

// The h buffer of a state is h [batch][E_k][N] fp32 followed by the fused decode path's x_proj
// accumulator [batch][hloc*P] fp32, which is all-zero between decode calls: the decode in_proj
// adds into it, decode_step reads it, out_proj's CTA 0 zeroes it again (at TP > 1 the AR#1
// publish kernel copies it out and re-zeroes it).
size_t xacc_offset(const ssm_tp_s* t, int batch) {
  return al256((size_t)batch * t->Ek * t->cfg.d_state * 4);
}
size_t h_total_bytes(const ssm_tp_s* t, int batch) {
  return xacc_offset(t, batch) + al256((size_t)batch * t->hloc * t->P * 4);
}

struct WsLayout {
  size_t xz, u, dbc, dlow, bc, delta, g, part, xn, xzf, uf, ssq, total;
};

// naive: + the all-gathered full-width activations of the SSM_TP_NAIVE arm (xz [M][2E], u [M][E])
WsLayout ws_layout(const ssm_tp_s* t, int64_t M, bool naive = false) {
  WsLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += al256(bytes); return o; };
  const size_t es = t->es;
  L.xz = take(M * 2 * t->Ek * es);
  L.u = take(M * t->Ek * es);
  L.dbc = take(M * t->hloc * t->P * 4);
  L.dlow = take((size_t)t->hloc * M * t->cfg.dt_rank * es);
  L.bc = take((size_t)t->hloc * M * 2 * t->cfg.d_state * 4);
  L.delta = take(M * t->Ek * es);
  L.g = take(M * t->Ek * es);
  L.part = take(t->k > 1 ? M * t->cfg.d_model * 4 : 0);
  L.xn = take(M * t->cfg.d_model * es);                  // pre-norm output (ssm_mixer_decode_block)
  L.xzf = take(naive ? M * 2 * t->cfg.d_inner * es : 0);
  L.uf = take(naive ? M * t->cfg.d_inner * es : 0);
  L.ssq = take(M * ((t->cfg.d_model + 31) / 32) * 4);    // out_proj row-chunk sums of squares (prefill_normed)
  L.total = off;
  return L;
}

size_t payload_bytes(const ssm_config_t* c, int k, int64_t M) {
  const int H = c->n_heads < 1 ? 1 : c->n_heads;
  const int hloc = H > k ? H / k : 1;
  const int P = c->dt_rank + 2 * c->d_state;
  size_t ar1 = (size_t)M * hloc * P * 4;
  size_t ar2q = al256((size_t)M * c->d_model) + (size_t)M * (c->d_model / (c->qar_block > 0 ? c->qar_block : 128)) * 4;
  size_t ar2f = (size_t)M * c->d_model * 4;
  const size_t es = c->dtype == SSM_BF16 ? 2 : 4;
  size_t agn = (size_t)M * 2 * (c->d_inner / k) * es;  // SSM_TP_NAIVE all-gather slices (in_proj, conv)
  size_t m = ar1 > ar2q ? ar1 : ar2q;
  if (agn > m) m = agn;
  return al256(m > ar2f ? m : ar2f);
}

size_t half_bytes(const ssm_tp_s* t) {
  if (t->buf_bytes <= kSigBytes) return 0;
  return ((t->buf_bytes - kSigBytes) / 2) & ~size_t(255);
}

ssm_status_t validate_cfg(const ssm_config_t* c, int k) {
  if (!c) return fail(SSM_ERR_ARG, "cfg is NULL");
  if (c->d_model <= 0 || c->d_inner <= 0 || c->d_state <= 0 || c->d_conv <= 0 || c->dt_rank <= 0)
    return fail(SSM_ERR_DIM, "non-positive dimension (d_model=%d d_inner=%d d_state=%d d_conv=%d dt_rank=%d)",
                c->d_model, c->d_inner, c->d_state, c->d_conv, c->dt_rank);
  if (c->dtype != SSM_BF16 && c->dtype != SSM_FP32) return fail(SSM_ERR_UNSUPPORTED, "dtype %d", c->dtype);
  if (c->d_state != 16 && c->d_state != 8) return fail(SSM_ERR_UNSUPPORTED, "d_state=%d (supported: 8, 16)", c->d_state);
  if (c->d_conv < 2 || c->d_conv > 4) return fail(SSM_ERR_UNSUPPORTED, "d_conv=%d (supported: 2..4)", c->d_conv);
  if (c->dt_rank + 2 * c->d_state > 320) return fail(SSM_ERR_UNSUPPORTED, "dt_rank + 2*d_state > 320");
  const int H = c->n_heads;
  if (H < 1 || c->d_inner % H) return fail(SSM_ERR_SHARD, "n_heads=%d does not divide d_inner=%d", H, c->d_inner);
  if (k < 1 || k > kMaxTP) return fail(SSM_ERR_UNSUPPORTED, "tp_size=%d (supported: 1..8)", k);
  if (c->d_inner % k) return fail(SSM_ERR_SHARD, "d_inner=%d not divisible by tp_size=%d", c->d_inner, k);
  if (H % k && k % H) return fail(SSM_ERR_SHARD, "n_heads=%d and tp_size=%d: heads cannot be split evenly", H, k);
  const int Ek = c->d_inner / k;
  if (Ek % 8) return fail(SSM_ERR_UNSUPPORTED, "d_inner/tp=%d must be a multiple of 8", Ek);
  const int cph = H > k ? Ek / (H / k) : Ek;
  if (cph % 32) return fail(SSM_ERR_UNSUPPORTED, "channels per local head (%d) must be a multiple of 32", cph);
  if (c->d_model % 16) return fail(SSM_ERR_UNSUPPORTED, "d_model=%d must be a multiple of 16", c->d_model);
  if (k > 1) {
    const int blk = c->qar_block;
    if (!(blk == 32 || blk == 64 || blk == 128 || blk == 256) || c->d_model % blk)
      return fail(SSM_ERR_UNSUPPORTED, "qar_block=%d must be 32/64/128/256 and divide d_model=%d", blk, c->d_model);
  }
  return SSM_OK;
}

cudaError_t gemm(ssm_tp_s* t, const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                 int ksplit, const Epilogue& e, cudaStream_t s, bool a_is_weight = false,
                 const void* a_blocked = nullptr) {
  t->launches++;
  if (t->bf16 && gemm_tc_supported(A, lda, B, ldb))
    return gemm_tc_bf16(reinterpret_cast<const __nv_bfloat16*>(A), lda, reinterpret_cast<const __nv_bfloat16*>(B),
                        ldb, M, N, K, ksplit, e, t->num_sms, s, a_is_weight && t_launch_pdl,
                        reinterpret_cast<const __nv_bfloat16*>(a_blocked));
  return gemm_simt(A, lda, B, ldb, t->bf16, M, N, K, ksplit, e, s);
}


// RAII probe: records an event pair around the launches in its scope when `kind` is probed.
struct Probe {
  ssm_tp_s* t;
  cudaStream_t s;
  int idx = -1;
  ssm_tp_s::ProbeSlot* slot = nullptr;
  Probe(ssm_tp_s* t_, int kind, cudaStream_t s_) : t(t_), s(s_) {
    if (kind < 0 || kind >= 16) return;
    ssm_tp_s::ProbeSlot& p = t->probes[kind];
    if (p.n >= p.cap) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) return;
    if (cs != cudaStreamCaptureStatusNone && kind != SSM_PROBE_IN_PROJ_DECODE) return;
    slot = &p;
    idx = p.n++;
    // inside a capture, an externally observable event-record node needs cudaEventRecordExternal
    flags = cs != cudaStreamCaptureStatusNone ? cudaEventRecordExternal : cudaEventRecordDefault;
    cudaEventRecordWithFlags(p.ev[2 * idx], s, flags);
  }
  ~Probe() {
    if (idx >= 0) cudaEventRecordWithFlags(slot->ev[2 * idx + 1], s, flags);
  }
  unsigned int flags = cudaEventRecordDefault;
};

// split-K factor for a swap-AB decode GEMM with `rows` weight rows and reduction length K:
// enough units to cover ~half the SMs, at least 4 k-blocks per unit
int split_for(const ssm_tp_s* t, int rows, int K) {
  const int tiles = (rows + 127) / 128;
  const int kb = (K + 63) / 64;
  int ks = t->num_sms / tiles;
  if (ks > kb) ks = kb;
  if (ks > 32) ks = 32;
  return ks < 1 ? 1 : ks;
}

Epilogue epi(int kind, int trans, void* C, int64_t ldc, const float* bias = nullptr) {
  Epilogue e{};
  e.kind = kind;
  e.trans = trans;
  e.C = C;
  e.ldc = ldc;
  e.bias = bias;
  return e;
}

Peers group_peers(const ssm_tp_s* t, int gsize) {
  Peers p{};
  const int g0 = (t->rank / gsize) * gsize;
  for (int i = 0; i < gsize; ++i) p.p[i] = t->peers.p[g0 + i];
  return p;
}

// One mixer layer. decode: seqlen == 1 path with in-place state update.
// norm_res != NULL (decode blocks): x_in = RMSNorm(norm_res) (weight 1, eps norm_eps; reading
// Q16) first, by the rmsnorm kernel.
ssm_status_t run_layer(ssm_tp_s* t, const ssm_layer_weights_t* w, ssm_state_s* st, const void* x_in, float* residual,
                       int batch, int seqlen, uint32_t flags, void* ws, bool decode, cudaStream_t s,
                       const float* norm_res = nullptr, float norm_eps = 0.f, const float* ss_in = nullptr,
                       void* x_next = nullptr, float* ss_next = nullptr) {
  // ss_in (prefill_normed): x_in is bf16(residual) itself and the in_proj epilogue applies the pre-norm
  // 1 / sqrt(ss_in / D + eps) per row; x_next / ss_next: the out_proj epilogue that adds into the
  // residual also writes bf16(new residual) and its row statistic for the next layer (reading Q22)
  const ssm_config_t& c = t->cfg;
  const int64_t M = (int64_t)batch * seqlen;
  const int D = c.d_model, Ek = t->Ek, R = c.dt_rank, N = c.d_state, K = c.d_conv, P = t->P, hl = t->hloc;
  const int bf = t->bf16;
  const bool naive = (flags & SSM_TP_NAIVE) != 0;
  const WsLayout L = ws_layout(t, M, naive);
  char* W = reinterpret_cast<char*>(ws);
  void* xz = W + L.xz;
  void* u = W + L.u;
  float* dbc = reinterpret_cast<float*>(W + L.dbc);
  void* dlow = W + L.dlow;
  float* BC = reinterpret_cast<float*>(W + L.bc);
  void* delta = W + L.delta;
  void* g = W + L.g;
  float* part = reinterpret_cast<float*>(W + L.part);
  const int kst = bf ? EPI_STORE_BF16 : EPI_STORE_F32;
  const int ksp = bf ? EPI_SOFTPLUS_BF16 : EPI_SOFTPLUS_F32;
  const bool swap = decode && bf;  // swap-AB: weights fill the 128-row MMA tile, batch is N
  const size_t es = t->es;
  const size_t half = half_bytes(t);
  auto own_half = [&](uint32_t ep) -> char* {
    return reinterpret_cast<char*>(t->peers.p[t->rank]) + kSigBytes + (ep & 1) * half;
  };
  auto half_off = [&](uint32_t ep) -> int64_t { return (int64_t)(kSigBytes + (ep & 1) * half); };

  const int64_t nD = M * D;
  // Collective epochs and destinations, fixed up front in execution order (AR#1 then AR#2).
  // Double buffering: collective e uses half e & 1.  A rank may write its half for collective e
  // only after its barrier of collective e - 1 has passed (every peer has then finished reading
  // the same half for collective e - 2), so no symmetric half is written before this layer's
  // first barrier except by the collective that barrier belongs to.
  const bool ar1 = t->ar1_group > 1;
  // SSM_TP_NAIVE: two all-gathers first (in_proj output, conv output), then AR#1 and AR#2
  const uint32_t ep_ag1 = naive ? ++t->epoch : 0, ep_ag2 = naive ? ++t->epoch : 0;
  const int E = c.d_inner, wn = 2 * E / t->k;  // naive: packed in_proj rows per rank
  if (naive) {
    t->ar_count += 2;
    t->bytes_sent += M * wn * es + M * Ek * es;
  }
  // packed [x ; z] activation: rank-local [M][2E_k] (channel split) or the gathered [M][2E] (naive)
  char* xzb = naive ? W + L.xzf : reinterpret_cast<char*>(xz);
  const int64_t ldxz = naive ? 2 * E : 2 * Ek;
  const int64_t xoff = naive ? (int64_t)t->rank * Ek : 0, zoff = naive ? E + (int64_t)t->rank * Ek : Ek;
  uint32_t ep1 = 0, ep2 = 0;
  float* xdst = dbc;
  if (ar1) {
    ep1 = ++t->epoch;
    xdst = reinterpret_cast<float*>(own_half(ep1));
    t->ar_count++;
    t->bytes_sent += M * hl * P * 4;
  }
  enum { OUT_RESID, OUT_EXTERNAL, OUT_FP32, OUT_INT8, OUT_W16 } omode;
  float* odst;
  if (t->k == 1) {
    omode = OUT_RESID;
    odst = residual;
  } else if (flags & SSM_AR2_EXTERNAL) {
    omode = OUT_EXTERNAL;
    odst = residual;
  } else if (flags & (SSM_AR2_FP16 | SSM_AR2_BF16)) {
    omode = OUT_W16;
    ep2 = ++t->epoch;
    odst = part;
  } else if (flags & SSM_AR2_FP32) {
    omode = OUT_FP32;
    ep2 = ++t->epoch;
    // decode: the split-K out_proj accumulates into the zeroed local partial (zeroed before this
    // layer's AR#1 barrier: it cannot be the symmetric half), copied over by the publish kernel;
    // prefill: stored straight into the half (the out_proj runs after the AR#1 barrier)
    odst = swap ? part : reinterpret_cast<float*>(own_half(ep2));
  } else {
    omode = OUT_INT8;
    ep2 = ++t->epoch;
    odst = part;
  }
  const bool oacc = omode == OUT_RESID;  // out_proj accumulates into its destination
  // int8 AR#2 schedule (reading Q6): two-shot with shared scales for k >= 4 and >= 64 tokens; the
  // requantised two-shot only on request (labelled variant)
  const bool requant = omode == OUT_INT8 && (flags & SSM_QAR_REQUANT) && nD % ((int64_t)t->k * c.qar_block) == 0;
  const bool twoshot = omode == OUT_INT8 && !requant &&
                       (flags & SSM_QAR_TWOSHOT || (!(flags & SSM_QAR_ONESHOT) && t->k >= 4 && M >= 64)) &&
                       nD % (16 * t->k) == 0 &&
                       2 * al256((size_t)nD / c.qar_block * 4) + al256(nD) + 2 * (size_t)nD / t->k <= half_bytes(t);
  // one-shot int8 at prefill: the out_proj epilogue quantises its TMEM accumulator straight into the
  // symmetric buffer (codes + per-block scales; no fp32 partial in HBM, no quantize kernel)
  const bool qfuse = omode == OUT_INT8 && !twoshot && !requant && !swap && bf && gemm_tc_supported(g, Ek, w->w_out, Ek);
  // decode GEMMs (swap-AB): split-K with the fp32 atomic epilogue so the few weight-row tiles
  // spread over the SMs (measured best: ~1 unit per SM, <= 32 splits)
  // (naive decode: no split-K for x_proj -- its zero-fill of the AR#1 half would precede the
  // all-gather barrier of the same half's previous use)
  const int ks_x = swap && !naive ? split_for(t, hl * P, Ek) : 1;
  const int ks_o = swap ? split_for(t, D, Ek) : 1;

  // (a1) in_proj, column-parallel: xz = x_in W_in,r^T   [M, 2E_k]
  // Fused decode: the in_proj epilogue also runs the conv step (a2) and adds its x_proj partial
  // (a3) into the state's zeroed accumulator (at TP > 1 published to the symmetric buffer by
  // publish_barrier_kernel, which is also AR#1's barrier).
  float* xacc = reinterpret_cast<float*>(reinterpret_cast<char*>(st->h) + xacc_offset(t, batch));
  const bool fuse = swap && !naive && !(flags & SSM_DECODE_UNFUSED) && batch <= 32 && P <= 320 && P % 2 == 0 && K >= 2 &&
                    K <= 4 && t->cph % 128 == 0 && gemm_tc_supported(w->w_in, D, x_in, D);
  if (norm_res) {
    t->launches++;
    CU(launch_rmsnorm(bf, norm_res, nullptr, norm_eps, const_cast<void*>(x_in), M, D, s));
  }
  {
    Probe pr(t, decode ? SSM_PROBE_IN_PROJ_DECODE : SSM_PROBE_IN_PROJ, s);
    if (fuse) {
      t->fused_calls++;
      Epilogue e = epi(EPI_DECODE_INPROJ, 1, xz, 2 * Ek);
      e.cst = st->conv;
      e.cw = w->conv_w;
      e.cb = w->conv_b;
      e.u = u;
      e.wx = w->w_x;
      e.xacc = xacc;
      e.Ek = Ek;
      e.K = K;
      e.P = P;
      e.hl = hl;
      e.cph = t->cph;
      if (!oacc) { e.zero = odst; e.nzero = nD; }  // out_proj partial target (local workspace)
      CU(gemm(t, w->w_in, D, x_in, D, 2 * Ek, (int)M, D, 1, e, s, true, w->w_in_pk));
    } else if (naive) {
      // (i) this rank's uniform slice of the packed in_proj -> own half, barrier, all-gather of the
      // full packed activation [x ; z] ("after the input projection")
      char* dst = own_half(ep_ag1);
      if (swap)
        CU(gemm(t, w->w_in_naive, D, x_in, D, wn, (int)M, D, 1, epi(kst, 1, dst, wn), s, true));
      else
        CU(gemm(t, x_in, D, w->w_in_naive, D, (int)M, wn, D, 1, epi(kst, 0, dst, wn), s));
      t->launches += 2;
      CU(launch_peer_barrier(t->peers, t->rank, t->k, s));
      CU(launch_gather_cols(t->peers, t->k, half_off(ep_ag1), M, (int)(wn * es), xzb, ldxz * (int64_t)es, s));
    } else if (swap)
      CU(gemm(t, w->w_in, D, x_in, D, 2 * Ek, (int)M, D, 1, epi(kst, 1, xz, 2 * Ek), s, true, w->w_in_pk));
    else {
      Epilogue e = epi(kst, 0, xz, 2 * Ek);
      if (ss_in) {
        e.rss = ss_in;
        e.rss_inv = 1.0f / (float)D;
        e.rss_eps = norm_eps;
      }
      CU(gemm(t, x_in, D, w->w_in, D, (int)M, 2 * Ek, D, 1, e, s));
    }
  }
  // naive: the conv output goes to this rank's half for the second all-gather
  if (naive) u = own_half(ep_ag2);

  // (a2) conv1d + SiLU, rank-local; conv window of the cache updated
  if (decode && !fuse) {
    // split-K targets of x_proj / out_proj are zeroed by the conv kernel (one launch fewer)
    float* z0 = nullptr;
    int64_t n0 = 0;
    float* z1 = nullptr;
    int64_t n1 = 0;
    if (ks_x != 1) { z0 = xdst; n0 = M * hl * P; }
    if (swap && !oacc) { z1 = odst; n1 = nD; }
    if ((n0 & 3) && n0) { CU(cudaMemsetAsync(z0, 0, n0 * 4, s)); n0 = 0; }
    if ((n1 & 3) && n1) { CU(cudaMemsetAsync(z1, 0, n1 * 4, s)); n1 = 0; }
    Probe pr(t, SSM_PROBE_CONV, s);
    t->launches++;
    CU(launch_conv_decode(bf, xzb + xoff * es, ldxz, st->conv, w->conv_w, w->conv_b, u, Ek, batch, Ek, K, z0, n0, z1,
                          n1, nullptr, s));
  } else if (!decode) {
    Probe pr(t, SSM_PROBE_CONV, s);
    t->launches += 2;
    CU(launch_conv1d_silu(bf, xzb + xoff * es, ldxz, st->conv, w->conv_w, w->conv_b, u, Ek, batch, seqlen, Ek, K, s));
    CU(launch_conv_state_update(bf, xzb + xoff * es, ldxz, st->conv, batch, seqlen, Ek, K, s));
  }
  // (ii) naive: barrier, all-gather of the full-width conv output ("around the
  // convolution branch"); the x_proj partial then reads this rank's slice of the gathered layout
  const void* ux = u;
  int64_t ldux = Ek;
  if (naive) {
    t->launches += 2;
    CU(launch_peer_barrier(t->peers, t->rank, t->k, s));
    CU(launch_gather_cols(t->peers, t->k, half_off(ep_ag2), M, (int)(Ek * es), W + L.uf, (int64_t)E * es, s));
    ux = W + L.uf + xoff * es;
    ldux = E;
  }

  // TP = 1 prefill without the Falcon dt/B/C RMSNorm: the x_proj epilogue writes the unpacked fields
  const bool split_dbc = bf && !decode && !swap && !ar1 && !naive && !c.bcdt_rmsnorm && R % 32 == 0 && P % 32 == 0 &&
                         gemm_tc_supported(ux, ldux, w->w_x, Ek);
  // (a3) x_proj partial [M, hloc*P] fp32, straight into the symmetric buffer when AR#1 follows
  if (!fuse) {
    Probe pr(t, SSM_PROBE_X_PROJ, s);
    if (swap)
      CU(gemm(t, w->w_x, Ek, ux, ldux, hl * P, (int)M, Ek, ks_x,
              epi(ks_x != 1 ? EPI_ATOMIC_F32 : EPI_STORE_F32, 1, xdst, hl * P), s, true, naive ? nullptr : w->w_x_pk));
    else if (split_dbc) {  // TP = 1: dt_low (bf16) and B || C (fp32) stored by the epilogue (no unpack pass)
      Epilogue e = epi(EPI_SPLIT_DBC, 0, xdst, hl * P);
      e.dbc_low = dlow;
      e.dbc_bc = BC;
      e.dbc_R = R;
      e.dbc_P = P;
      e.dbc_M = (int)M;
      CU(gemm(t, ux, ldux, w->w_x, Ek, (int)M, hl * P, Ek, 1, e, s));
    } else
      CU(gemm(t, ux, ldux, w->w_x, Ek, (int)M, hl * P, Ek, 1, epi(EPI_STORE_F32, 0, xdst, hl * P), s));
  }

  // (a4) AR#1: barrier, then the fixed-order sum is done by its consumer
  Peers dsrc{};
  int nsrc = 1;
  int64_t doff = 0;
  if (ar1) {
    t->launches++;
    if (fuse)
      CU(launch_publish_barrier(t->peers, t->rank, t->k, xacc, (int64_t)batch * hl * P, half_off(ep1), s));
    else
      CU(launch_peer_barrier(t->peers, t->rank, t->k, s));
    dsrc = group_peers(t, t->ar1_group);
    nsrc = t->ar1_group;
    doff = half_off(ep1);
  } else {
    dsrc.p[0] = fuse ? xacc : dbc;
  }

  if (decode) {
    // (a4)-(a7) decode: AR#1 sum + unpack + dt_proj + softplus + scan step + gate, one kernel
    Probe pr(t, SSM_PROBE_DECODE_STEP, s);
    t->launches++;
    CU(launch_decode_step(bf, dsrc, nsrc, doff, hl * P, c.bcdt_rmsnorm, c.rms_eps, u, xzb + zoff * es, ldxz, w->w_dt,
                          w->b_dt, w->a_log, w->d_skip, st->h, g, batch, Ek, R, N, t->cph, nullptr, s));
  } else {
    // (a4) unpack dt_low / B / C (unless the x_proj epilogue split them); (a5) dt_proj + softplus;
    // (a6)+(a7) scan, D skip, gate
    if (!split_dbc) {
      t->launches++;
      CU(launch_unpack(bf, dsrc, nsrc, doff, (int)M, hl, R, N, c.bcdt_rmsnorm, c.rms_eps, dlow, BC, s));
    }
    {
      Probe pr(t, SSM_PROBE_DT_PROJ, s);
      for (int j = 0; j < hl; ++j) {
        const int c0 = j * t->cph;
        const char* dl_j = reinterpret_cast<const char*>(dlow) + (size_t)j * M * R * es;
        CU(gemm(t, dl_j, R, reinterpret_cast<const char*>(w->w_dt) + (size_t)c0 * R * es, R, (int)M, t->cph, R, 1,
                epi(ksp, 0, reinterpret_cast<char*>(delta) + c0 * es, Ek, w->b_dt + c0), s));
      }
    }
    Probe pr(t, SSM_PROBE_SCAN, s);
    for (int j = 0; j < hl; ++j) {
      const int c0 = j * t->cph;
      t->launches++;
      CU(launch_scan(bf, bf, reinterpret_cast<char*>(u) + c0 * es, Ek, reinterpret_cast<char*>(delta) + c0 * es, Ek,
                     xzb + (zoff + c0) * es, ldxz, BC + (size_t)j * M * 2 * N, 2 * N,
                     w->a_log + (size_t)c0 * N, w->d_skip + c0, st->h + (size_t)c0 * N, (int64_t)Ek * N,
                     reinterpret_cast<char*>(g) + c0 * es, Ek, batch, seqlen, t->cph, N, s));
    }
  }

  // (a8) out_proj, row-parallel partial (TP=1: added straight into the fp32 residual)
  {
    Probe pr(t, SSM_PROBE_OUT_PROJ, s);
    if (swap) {
      Epilogue e = epi(EPI_ATOMIC_F32, 1, odst, D);
      // re-arm the x_proj accumulator (at TP > 1 the publish kernel re-zeroes it)
      if (fuse && !ar1) { e.zero = xacc; e.nzero = (int64_t)batch * hl * P; }
      CU(gemm(t, w->w_out, Ek, g, Ek, D, (int)M, Ek, ks_o, e, s, true, w->w_out_pk));
    } else if (qfuse) {
      Epilogue e = epi(EPI_QUANT_I8, 0, own_half(ep2), D);
      e.qs = reinterpret_cast<float*>(own_half(ep2) + al256(nD));
      e.qblk = c.qar_block;
      CU(gemm(t, g, Ek, w->w_out, Ek, (int)M, D, Ek, 1, e, s));
    } else {
      Epilogue e = epi(oacc ? EPI_ADD_F32 : EPI_STORE_F32, 0, odst, D);
      if (x_next && t->k == 1) {
        e.cpy = x_next;
        e.ssq = reinterpret_cast<float*>(W + L.ssq);
      }
      CU(gemm(t, g, Ek, w->w_out, Ek, (int)M, D, Ek, 1, e, s));
      if (x_next && t->k == 1) {
        t->launches++;
        CU(launch_ssq_finalize(reinterpret_cast<float*>(W + L.ssq), (D + 31) / 32, ss_next, M, s));
      }
    }
  }
  // (a9) AR#2 at the residual boundary
  if (omode == OUT_FP32) {
    Probe pr(t, SSM_PROBE_AR2, s);
    t->ar_count++;
    t->bytes_sent += nD * 4;
    t->launches += 2;
    if (swap)  // local partial -> own half (re-zeroing the partial), then the barrier
      CU(launch_publish_barrier(t->peers, t->rank, t->k, part, nD, half_off(ep2), s));
    else
      CU(launch_peer_barrier(t->peers, t->rank, t->k, s));
    CU(launch_f32_reduce(t->peers, t->k, half_off(ep2), nD, residual, 1, s));
  } else if (omode == OUT_W16) {  // the paper's FP32 -> FP16 wire or the bf16 arm
    Probe pr(t, SSM_PROBE_AR2, s);
    const int wbf = (flags & SSM_AR2_BF16) ? 1 : 0;
    t->launches += 3;
    CU(launch_w16_cast(wbf, part, nD, own_half(ep2), s));
    t->ar_count++;
    t->bytes_sent += nD * 2;
    CU(launch_peer_barrier(t->peers, t->rank, t->k, s));
    CU(launch_w16_reduce(wbf, t->peers, t->k, half_off(ep2), nD, residual, 1, s));
  } else if (requant) {  // requantised two-shot (labelled variant of reading Q6)
    Probe pr(t, SSM_PROBE_AR2, s);
    t->launches += 5;
    t->ar_count++;
    t->bytes_sent += 2 * (nD + nD / c.qar_block * 4) * (t->k - 1) / t->k;
    CU(launch_qar_requant(t->peers, t->rank, t->k, half_off(ep2), part, nD, c.qar_block, residual, 1, s));
  } else if (twoshot) {
    // two-shot schedule with shared scales (reading Q6): (k-1)/k 3n B on the wire instead of (k-1) n
    Probe pr(t, SSM_PROBE_AR2, s);
    t->launches += 7;
    t->ar_count++;
    t->bytes_sent += (nD + 2 * nD / t->k) * (t->k - 1) / t->k + nD / c.qar_block * 4;
    CU(launch_qar_twoshot(t->peers, t->rank, t->k, half_off(ep2), part, nD, c.qar_block, residual, 1, s, x_next,
                          x_next ? reinterpret_cast<float*>(W + L.ssq) : nullptr, D));
  } else if (omode == OUT_INT8) {
    Probe pr(t, SSM_PROBE_AR2, s);
    int8_t* q = reinterpret_cast<int8_t*>(own_half(ep2));
    float* sc = reinterpret_cast<float*>(own_half(ep2) + al256(nD));
    t->launches += qfuse ? 2 : 3;
    if (!qfuse) CU(launch_quantize(part, nD, c.qar_block, q, sc, s));
    t->ar_count++;
    t->bytes_sent += nD + nD / c.qar_block * 4;
    CU(launch_peer_barrier(t->peers, t->rank, t->k, s));
    CU(launch_qar_reduce(t->peers, t->k, half_off(ep2), half_off(ep2) + (int64_t)al256(nD), nD, c.qar_block, residual,
                         1, s, x_next, x_next ? reinterpret_cast<float*>(W + L.ssq) : nullptr, D));
  }
  // TP > 1 with the pre-norm folded (prefill_normed): the AR#2 kernel that finished the residual rows
  // wrote their bf16 copy and per-chunk sums of squares; the row statistic for the next in_proj
  if (x_next && t->k > 1) {
    t->launches++;
    CU(launch_ssq_finalize(reinterpret_cast<float*>(W + L.ssq), (D + 31) / 32, ss_next, M, s));
  }
  return SSM_OK;
}

ssm_status_t check_call(ssm_tp_s* t, const ssm_layer_weights_t* w, ssm_state_s* st, const void* x_in,
                        const float* residual, int batch, int seqlen, uint32_t flags, void* ws, size_t ws_bytes) {
  if (!t) return fail(SSM_ERR_ARG, "tp handle is NULL");
  if (!w || !w->w_in || !w->conv_w || !w->conv_b || !w->w_x || !w->w_dt || !w->b_dt || !w->a_log || !w->d_skip ||
      !w->w_out)
    return fail(SSM_ERR_ARG, "weights struct or one of its pointers is NULL");
  if (!st) return fail(SSM_ERR_ARG, "state is NULL");
  if (st->owner != t) return fail(SSM_ERR_CACHE, "state belongs to another handle");
  if (st->batch != batch) return fail(SSM_ERR_CACHE, "state batch %d != call batch %d", st->batch, batch);
  if (batch < 0 || seqlen < 0) return fail(SSM_ERR_DIM, "negative batch/seqlen");
  if (!x_in || !residual) return fail(SSM_ERR_ARG, "x_in/residual is NULL");
  if ((reinterpret_cast<uintptr_t>(x_in) | reinterpret_cast<uintptr_t>(residual)) & 15)
    return fail(SSM_ERR_ARG, "x_in/residual must be 16-B aligned");
  if (flags & ~(uint32_t)(SSM_AR2_INT8 | SSM_AR2_FP16 | SSM_AR2_BF16 | SSM_AR2_FP32 | SSM_AR2_EXTERNAL |
                          SSM_QAR_TWOSHOT | SSM_QAR_ONESHOT | SSM_QAR_REQUANT | SSM_DECODE_UNFUSED | SSM_TP_NAIVE))
    return fail(SSM_ERR_ARG, "unknown flags 0x%x", flags);
  if ((flags & SSM_QAR_TWOSHOT) && (flags & SSM_QAR_ONESHOT))
    return fail(SSM_ERR_ARG, "SSM_QAR_TWOSHOT and SSM_QAR_ONESHOT are exclusive");
  const int nmode = !!(flags & SSM_AR2_INT8) + !!(flags & SSM_AR2_FP16) + !!(flags & SSM_AR2_BF16) + !!(flags & SSM_AR2_FP32) +
                    !!(flags & SSM_AR2_EXTERNAL);
  if (nmode > 1) return fail(SSM_ERR_ARG, "at most one AR#2 mode flag");
  const int64_t M = (int64_t)batch * seqlen;
  const bool naive = (flags & SSM_TP_NAIVE) != 0;
  if (naive && (t->k < 2 || t->hloc != 1 || t->ar1_group < 2 || !w->w_in_naive))
    return fail(SSM_ERR_UNSUPPORTED, "SSM_TP_NAIVE needs tp_size > 1, one x_proj head per rank and w_in_naive");
  const WsLayout L = ws_layout(t, M, naive);
  if (M > 0 && (!ws || ws_bytes < L.total))
    return fail(SSM_ERR_ARG, "workspace %zu B < required %zu B", ws_bytes, L.total);
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(SSM_ERR_ARG, "workspace must be 256-B aligned");
  if (t->k > 1 && !(flags & SSM_AR2_EXTERNAL) && payload_bytes(&t->cfg, t->k, M) > half_bytes(t))
    return fail(SSM_ERR_ARG, "symmetric buffer (%zu B) too small for %lld tokens (need %zu B)", t->buf_bytes,
                (long long)M, kSigBytes + 2 * payload_bytes(&t->cfg, t->k, M));
  return SSM_OK;
}

}  // namespace

extern "C" {

const char* ssm_last_error(void) { return g_err.c_str(); }
const char* ssm_version(void) { return "libssmtp 0.1 (sm_100a)"; }

ssm_status_t ssm_tp_init(const ssm_config_t* cfg, const ssm_comm_t* comm, ssm_tp_t* out) {
  if (!out) return fail(SSM_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!comm) return fail(SSM_ERR_ARG, "comm is NULL");
  const int k = comm->tp_size;
  if (k < 1 || k > kMaxTP) return fail(SSM_ERR_UNSUPPORTED, "tp_size=%d (supported: 1..8)", k);
  if (comm->rank < 0 || comm->rank >= k) return fail(SSM_ERR_RANK, "rank %d not in [0,%d)", comm->rank, k);
  ssm_status_t st = validate_cfg(cfg, k);
  if (st != SSM_OK) return st;
  if (k > 1) {
    if (!comm->peer_bufs) return fail(SSM_ERR_ARG, "peer_bufs is NULL with tp_size=%d", k);
    for (int i = 0; i < k; ++i)
      if (!comm->peer_bufs[i] || (reinterpret_cast<uintptr_t>(comm->peer_bufs[i]) & 255))
        return fail(SSM_ERR_ARG, "peer_bufs[%d] is NULL or not 256-B aligned", i);
    if (comm->buf_bytes < kSigBytes + 2 * payload_bytes(cfg, k, 1))
      return fail(SSM_ERR_ARG, "buf_bytes=%zu too small", comm->buf_bytes);
  }
  ssm_tp_s* t = new (std::nothrow) ssm_tp_s();
  if (!t) return fail(SSM_ERR_ARG, "out of host memory");
  t->cfg = *cfg;
  if (t->cfg.qar_block <= 0) t->cfg.qar_block = 128;
  t->rank = comm->rank;
  t->k = k;
  t->flags = comm->flags;
  for (int i = 0; i < k && comm->peer_bufs; ++i) t->peers.p[i] = comm->peer_bufs[i];
  t->buf_bytes = comm->buf_bytes;
  const int H = cfg->n_heads;
  t->Ek = cfg->d_inner / k;
  t->P = cfg->dt_rank + 2 * cfg->d_state;
  t->hloc = H > k ? H / k : 1;
  t->cph = t->Ek / t->hloc;
  t->ar1_group = k > H ? k / H : 1;
  t->bf16 = cfg->dtype == SSM_BF16;
  t->es = t->bf16 ? 2 : 4;
  t->epoch = 0;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) {
    t->num_sms = sms;
    static std::once_flag once;
    static cudaError_t pre = cudaSuccess;
    std::call_once(once, [] {
      pre = preload_kernels();
      if (pre == cudaSuccess) pre = preload_gemm_simt();
      if (pre == cudaSuccess) pre = preload_gemm_tc();
      if (pre == cudaSuccess) pre = preload_attn();
      if (pre == cudaSuccess) pre = preload_ssd();
      if (pre == cudaSuccess) pre = preload_decode_stack();
    });
    if (pre != cudaSuccess) {
      delete t;
      return fail(SSM_ERR_CUDA, "kernel preload failed: %s", cudaGetErrorString(pre));
    }
  } else {
    cudaGetLastError();
    t->num_sms = 148;
  }
  *out = t;
  return SSM_OK;
}

ssm_status_t ssm_tp_destroy(ssm_tp_t tp) {
  if (tp)
    for (int k = 0; k < 16; ++k) ssm_tp_probe(tp, k, 0);
  delete tp;
  return SSM_OK;
}

ssm_status_t ssm_tp_probe(ssm_tp_t tp, int32_t kernel, int32_t capacity) {
  if (!tp) return fail(SSM_ERR_ARG, "tp is NULL");
  if (capacity < 0) return fail(SSM_ERR_ARG, "capacity < 0");
  if (kernel < 0 || kernel >= 16) return fail(SSM_ERR_ARG, "kernel id %d", kernel);
  ssm_tp_s::ProbeSlot& p = tp->probes[kernel];
  if (p.ev) {
    for (int i = 0; i < 2 * p.cap; ++i) cudaEventDestroy(p.ev[i]);
    delete[] p.ev;
    p.ev = nullptr;
  }
  p.cap = 0;
  p.n = 0;
  if (capacity == 0) return SSM_OK;
  p.ev = new (std::nothrow) cudaEvent_t[2 * capacity];
  if (!p.ev) return fail(SSM_ERR_ARG, "out of host memory");
  for (int i = 0; i < 2 * capacity; ++i) CU(cudaEventCreate(&p.ev[i]));
  p.cap = capacity;
  return SSM_OK;
}

ssm_status_t ssm_tp_probe_read(ssm_tp_t tp, int32_t kernel, float* ms, int32_t capacity, int32_t* n) {
  if (!tp || !n) return fail(SSM_ERR_ARG, "NULL argument");
  if (kernel < 0 || kernel >= 16) return fail(SSM_ERR_ARG, "kernel id %d", kernel);
  ssm_tp_s::ProbeSlot& p = tp->probes[kernel];
  const int cnt = p.n < capacity ? p.n : capacity;
  for (int i = 0; i < cnt; ++i) {
    CU(cudaEventSynchronize(p.ev[2 * i + 1]));
    CU(cudaEventElapsedTime(&ms[i], p.ev[2 * i], p.ev[2 * i + 1]));
  }
  *n = cnt;
  return SSM_OK;
}

ssm_status_t ssm_comm_bytes(const ssm_config_t* cfg, int32_t tp_size, int64_t max_tokens, size_t* bytes) {
  if (!bytes) return fail(SSM_ERR_ARG, "bytes is NULL");
  ssm_status_t st = validate_cfg(cfg, tp_size);
  if (st != SSM_OK) return st;
  if (max_tokens < 1) max_tokens = 1;
  *bytes = kSigBytes + 2 * payload_bytes(cfg, tp_size, max_tokens);
  return SSM_OK;
}

ssm_status_t ssm_workspace_bytes(ssm_tp_t tp, int32_t batch, int32_t seqlen, size_t* bytes) {
  if (!tp || !bytes) return fail(SSM_ERR_ARG, "NULL argument");
  if (batch < 0 || seqlen < 0) return fail(SSM_ERR_DIM, "negative batch/seqlen");
  *bytes = ws_layout(tp, (int64_t)batch * seqlen).total;
  return SSM_OK;
}

ssm_status_t ssm_workspace_bytes_flags(ssm_tp_t tp, int32_t batch, int32_t seqlen, uint32_t flags, size_t* bytes) {
  if (!tp || !bytes) return fail(SSM_ERR_ARG, "NULL argument");
  if (batch < 0 || seqlen < 0) return fail(SSM_ERR_DIM, "negative batch/seqlen");
  *bytes = ws_layout(tp, (int64_t)batch * seqlen, (flags & SSM_TP_NAIVE) != 0).total;
  return SSM_OK;
}

ssm_status_t ssm_state_bytes(ssm_tp_t tp, int32_t batch, size_t* conv_bytes, size_t* h_bytes) {
  if (!tp || !conv_bytes || !h_bytes) return fail(SSM_ERR_ARG, "NULL argument");
  if (batch < 1) return fail(SSM_ERR_DIM, "batch=%d", batch);
  *conv_bytes = (size_t)batch * (tp->cfg.d_conv - 1) * tp->Ek * tp->es;
  *h_bytes = h_total_bytes(tp, batch);
  return SSM_OK;
}

ssm_status_t ssm_state_alloc(ssm_tp_t tp, int32_t batch, void* conv_buf, size_t conv_bytes, void* h_buf,
                             size_t h_bytes, void* stream, ssm_state_t* out) {
  if (!out) return fail(SSM_ERR_ARG, "out is NULL");
  *out = nullptr;
  size_t cb = 0, hb = 0;
  ssm_status_t s = ssm_state_bytes(tp, batch, &cb, &hb);
  if (s != SSM_OK) return s;
  if (!conv_buf || !h_buf) return fail(SSM_ERR_ARG, "state buffers are NULL");
  if (conv_bytes < cb || h_bytes < hb)
    return fail(SSM_ERR_ARG, "state buffers too small (%zu/%zu B, need %zu/%zu B)", conv_bytes, h_bytes, cb, hb);
  if ((reinterpret_cast<uintptr_t>(conv_buf) | reinterpret_cast<uintptr_t>(h_buf)) & 15)
    return fail(SSM_ERR_ARG, "state buffers must be 16-B aligned");
  ssm_state_s* st = new (std::nothrow) ssm_state_s();
  if (!st) return fail(SSM_ERR_ARG, "out of host memory");
  st->owner = tp;
  st->batch = batch;
  st->conv = conv_buf;
  st->h = reinterpret_cast<float*>(h_buf);
  cudaStream_t s_ = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(conv_buf, 0, cb, s_) != cudaSuccess || cudaMemsetAsync(h_buf, 0, hb, s_) != cudaSuccess) {
    delete st;
    return fail(SSM_ERR_CUDA, "zero-fill of the state failed: %s", cudaGetErrorString(cudaGetLastError()));
  }
  *out = st;
  return SSM_OK;
}

ssm_status_t ssm_state_reset(ssm_state_t st, void* stream) {
  if (!st) return fail(SSM_ERR_ARG, "state is NULL");
  size_t cb = 0, hb = 0;
  ssm_state_bytes(st->owner, st->batch, &cb, &hb);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CU(cudaMemsetAsync(st->conv, 0, cb, s));
  CU(cudaMemsetAsync(st->h, 0, hb, s));
  return SSM_OK;
}

ssm_status_t ssm_state_free(ssm_state_t st) {
  delete st;
  return SSM_OK;
}

ssm_status_t ssm_mixer_prefill(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st, const void* x_in,
                               float* residual, int32_t batch, int32_t seqlen, uint32_t flags, void* workspace,
                               size_t ws_bytes, void* stream) {
  ssm_status_t s = check_call(tp, w, st, x_in, residual, batch, seqlen, flags, workspace, ws_bytes);
  if (s != SSM_OK) return s;
  if ((int64_t)batch * seqlen == 0) return SSM_OK;
  return run_layer(tp, w, st, x_in, residual, batch, seqlen, flags, workspace, false,
                   reinterpret_cast<cudaStream_t>(stream));
}

ssm_status_t ssm_mixer_prefill_normed(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st, const void* x_in,
                                      const float* ss_in, float norm_eps, float* residual, void* x_next,
                                      float* ss_next, int32_t batch, int32_t seqlen, uint32_t flags, void* workspace,
                                      size_t ws_bytes, void* stream) {
  ssm_status_t s = check_call(tp, w, st, x_in, residual, batch, seqlen, flags, workspace, ws_bytes);
  if (s != SSM_OK) return s;
  if (!ss_in || ((x_next == nullptr) != (ss_next == nullptr))) return fail(SSM_ERR_ARG, "ss_in NULL, or x_next / ss_next not both set");
  if (!(norm_eps >= 0.f)) return fail(SSM_ERR_ARG, "norm_eps must be >= 0");
  const int D = tp->cfg.d_model, Ek = tp->Ek;
  // the residual (and, with x_next, the next layer's pre-norm inputs) is finished by this rank's out_proj
  // epilogue at TP = 1 and by the int8 AR#2's reduce / all-gather kernel at TP > 1 (one-shot or
  // two-shot schedule); both projections on the tcgen05 GEMM
  const bool ar2_int8 = (flags & SSM_AR2_INT8) || !(flags & (SSM_AR2_FP16 | SSM_AR2_BF16 | SSM_AR2_FP32 | SSM_AR2_EXTERNAL));
  if ((tp->k > 1 && (!ar2_int8 || (flags & SSM_QAR_REQUANT) || D % 32)) || !tp->bf16 || (flags & SSM_TP_NAIVE) ||
      D % 8 || !gemm_tc_supported(x_in, D, w->w_in, D) || !gemm_tc_supported(w->w_out, Ek, w->w_out, Ek))
    return fail(SSM_ERR_UNSUPPORTED,
                "prefill_normed: bf16, tcgen05-compatible strides, and at TP > 1 the int8 AR#2 (one- or two-shot)");
  if ((reinterpret_cast<uintptr_t>(x_next) & 15) || ((reinterpret_cast<uintptr_t>(ss_in) | reinterpret_cast<uintptr_t>(ss_next)) & 3))
    return fail(SSM_ERR_ARG, "x_next must be 16-B aligned, ss_in / ss_next 4-B aligned");
  if ((int64_t)batch * seqlen == 0) return SSM_OK;
  return run_layer(tp, w, st, x_in, residual, batch, seqlen, flags, workspace, false,
                   reinterpret_cast<cudaStream_t>(stream), nullptr, norm_eps, ss_in, x_next, ss_next);
}

ssm_status_t ssm_rowstats(ssm_tp_t tp, const float* residual, void* x_out, float* ss_out, int64_t M, void* stream) {
  if (!tp || !residual || !x_out || !ss_out) return fail(SSM_ERR_ARG, "NULL argument");
  if (!tp->bf16) return fail(SSM_ERR_UNSUPPORTED, "ssm_rowstats: bf16 handles only");
  if ((reinterpret_cast<uintptr_t>(residual) | reinterpret_cast<uintptr_t>(x_out)) & 15)
    return fail(SSM_ERR_ARG, "pointers must be 16-B aligned");
  tp->launches++;
  CU(launch_rowstats(residual, x_out, ss_out, M, tp->cfg.d_model, reinterpret_cast<cudaStream_t>(stream)));
  return SSM_OK;
}

ssm_status_t ssm_mixer_decode(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st, const void* x_in,
                              float* residual, int32_t batch, uint32_t flags, void* workspace, size_t ws_bytes,
                              void* stream) {
  ssm_status_t s = check_call(tp, w, st, x_in, residual, batch, 1, flags, workspace, ws_bytes);
  if (s != SSM_OK) return s;
  if (batch == 0) return SSM_OK;
  // no PDL across virtual ranks: early-launched dependents of one rank's stream would hold the SMs
  // the other ranks' kernels need to reach the shared barrier
  PdlScope pdl(!(tp->flags & SSM_COMM_VIRTUAL));
  return run_layer(tp, w, st, x_in, residual, batch, 1, flags, workspace, true,
                   reinterpret_cast<cudaStream_t>(stream));
}

ssm_status_t ssm_mixer_decode_block(ssm_tp_t tp, const ssm_layer_weights_t* w, ssm_state_t st, float* residual,
                                    int32_t batch, float norm_eps, uint32_t flags, void* workspace, size_t ws_bytes,
                                    void* stream) {
  ssm_status_t s = check_call(tp, w, st, residual, residual, batch, 1, flags, workspace, ws_bytes);
  if (s != SSM_OK) return s;
  if (!(norm_eps >= 0.f)) return fail(SSM_ERR_ARG, "norm_eps must be >= 0");
  if (batch == 0) return SSM_OK;
  PdlScope pdl(!(tp->flags & SSM_COMM_VIRTUAL));
  void* xn = reinterpret_cast<char*>(workspace) + ws_layout(tp, batch).xn;
  return run_layer(tp, w, st, xn, residual, batch, 1, flags, workspace, true, reinterpret_cast<cudaStream_t>(stream),
                   residual, norm_eps);
}

ssm_status_t ssm_qallreduce(ssm_tp_t tp, const float* partial, float* out, size_t n, uint32_t flags, void* stream) {
  if (!tp) return fail(SSM_ERR_ARG, "tp is NULL");
  const uint32_t known = SSM_QAR_ACCUMULATE | SSM_QAR_FP16 | SSM_QAR_BF16 | SSM_QAR_TWOSHOT | SSM_QAR_REQUANT |
                         SSM_QAR_FP32;
  if (n == 0 && !(flags & ~known)) return SSM_OK;  // nothing to reduce
  if (!partial || !out) return fail(SSM_ERR_ARG, "NULL argument");
  if (flags & ~known) return fail(SSM_ERR_ARG, "unknown flags 0x%x", flags);
  if ((flags & SSM_QAR_FP16) && (flags & SSM_QAR_BF16)) return fail(SSM_ERR_ARG, "SSM_QAR_FP16 and SSM_QAR_BF16 are exclusive");
  const int blk = tp->cfg.qar_block;
  if (n % blk && !(flags & (SSM_QAR_FP32 | SSM_QAR_FP16 | SSM_QAR_BF16)))
    return fail(SSM_ERR_DIM, "n=%zu not a multiple of qar_block=%d", n, blk);
  if ((reinterpret_cast<uintptr_t>(partial) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(SSM_ERR_ARG, "pointers must be 16-B aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool acc = flags & SSM_QAR_ACCUMULATE;
  if (n == 0) return SSM_OK;
  if (tp->k == 1) {  // reading Q13: no quantisation at TP=1
    Peers one{};
    one.p[0] = const_cast<float*>(partial);
    tp->launches++;
    CU(launch_f32_reduce(one, 1, 0, (int64_t)n, out, acc, s));
    return SSM_OK;
  }
  if (flags & SSM_QAR_FP32) {  // exact: partial -> own half, barrier, fixed-order fp32 sum
    if (n % 4 || (reinterpret_cast<uintptr_t>(partial) & 15)) return fail(SSM_ERR_DIM, "n=%zu not a multiple of 4", n);
    if (n * 4 > half_bytes(tp)) return fail(SSM_ERR_ARG, "symmetric buffer too small for n=%zu", n);
    const uint32_t ep = ++tp->epoch;
    const int64_t off = (int64_t)(kSigBytes + (ep & 1) * half_bytes(tp));
    tp->launches += 2;
    tp->ar_count++;
    tp->bytes_sent += n * 4;
    CU(cudaMemcpyAsync(reinterpret_cast<char*>(tp->peers.p[tp->rank]) + off, partial, n * 4, cudaMemcpyDeviceToDevice, s));
    CU(launch_peer_barrier(tp->peers, tp->rank, tp->k, s));
    CU(launch_f32_reduce(tp->peers, tp->k, off, (int64_t)n, out, acc, s));
    return SSM_OK;
  }
  if (flags & SSM_QAR_REQUANT) {  // requantised two-shot int8 (labelled variant of reading Q6)
    if (n % ((size_t)tp->k * blk) || blk % 16) return fail(SSM_ERR_DIM, "n=%zu not a multiple of tp_size*qar_block", n);
    if (al256(n) + al256(n / blk * 4) + al256(n / tp->k) + n / tp->k / blk * 4 > half_bytes(tp))
      return fail(SSM_ERR_ARG, "symmetric buffer too small for n=%zu", n);
    const uint32_t ep = ++tp->epoch;
    tp->launches += 5;
    tp->ar_count++;
    tp->bytes_sent += 2 * (n + n / blk * 4) * (tp->k - 1) / tp->k;
    CU(launch_qar_requant(tp->peers, tp->rank, tp->k, (int64_t)(kSigBytes + (ep & 1) * half_bytes(tp)), partial,
                          (int64_t)n, blk, out, acc, s));
    return SSM_OK;
  }
  if (flags & SSM_QAR_TWOSHOT) {  // shared-scale two-shot int8 (reading Q6)
    if (n % (16 * (size_t)tp->k) || blk % 16) return fail(SSM_ERR_DIM, "n=%zu not a multiple of 16*tp_size", n);
    if (2 * al256(n / blk * 4) + al256(n) + 2 * n / tp->k > half_bytes(tp))
      return fail(SSM_ERR_ARG, "symmetric buffer too small for n=%zu", n);
    const uint32_t ep = ++tp->epoch;
    tp->launches += 7;
    tp->ar_count++;
    tp->bytes_sent += (n + 2 * n / tp->k) * (tp->k - 1) / tp->k + n / blk * 4;
    CU(launch_qar_twoshot(tp->peers, tp->rank, tp->k, (int64_t)(kSigBytes + (ep & 1) * half_bytes(tp)), partial,
                          (int64_t)n, blk, out, acc, s));
    return SSM_OK;
  }
  if (flags & (SSM_QAR_FP16 | SSM_QAR_BF16)) {  // the paper's fp16 wire / the bf16 arm
    const int wbf = (flags & SSM_QAR_BF16) ? 1 : 0;
    if (n % 8) return fail(SSM_ERR_DIM, "n=%zu not a multiple of 8 (fp16 wire)", n);
    if (n * 2 > half_bytes(tp)) return fail(SSM_ERR_ARG, "symmetric buffer too small for n=%zu", n);
    const uint32_t ep = ++tp->epoch;
    const size_t half = half_bytes(tp);
    char* own = reinterpret_cast<char*>(tp->peers.p[tp->rank]) + kSigBytes + (ep & 1) * half;
    tp->launches += 3;
    CU(launch_w16_cast(wbf, partial, (int64_t)n, own, s));
    tp->ar_count++;
    tp->bytes_sent += n * 2;
    CU(launch_peer_barrier(tp->peers, tp->rank, tp->k, s));
    CU(launch_w16_reduce(wbf, tp->peers, tp->k, (int64_t)(kSigBytes + (ep & 1) * half), (int64_t)n, out, acc, s));
    return SSM_OK;
  }
  const size_t need = al256(n) + n / blk * 4;
  if (need > half_bytes(tp)) return fail(SSM_ERR_ARG, "symmetric buffer too small for n=%zu", n);
  const uint32_t ep = ++tp->epoch;
  const size_t half = half_bytes(tp);
  char* own = reinterpret_cast<char*>(tp->peers.p[tp->rank]) + kSigBytes + (ep & 1) * half;
  const int64_t off = (int64_t)(kSigBytes + (ep & 1) * half);
  tp->launches += 3;
  CU(launch_quantize(partial, (int64_t)n, blk, reinterpret_cast<int8_t*>(own), reinterpret_cast<float*>(own + al256(n)), s));
  tp->ar_count++;
  tp->bytes_sent += n + n / blk * 4;
  CU(launch_peer_barrier(tp->peers, tp->rank, tp->k, s));
  CU(launch_qar_reduce(tp->peers, tp->k, off, off + (int64_t)al256(n), (int64_t)n, blk, out, acc, s));
  return SSM_OK;
}

ssm_status_t ssm_rmsnorm(ssm_tp_t tp, const float* residual, const float* weight, float eps, void* x_out, int64_t M,
                         void* stream) {
  if (!tp || !residual || !x_out) return fail(SSM_ERR_ARG, "NULL argument");
  // decode-sized rows: overlap with the neighbours (not across virtual ranks, see ssm_mixer_decode)
  PdlScope pdl(M <= 256 && !(tp->flags & SSM_COMM_VIRTUAL));
  if ((reinterpret_cast<uintptr_t>(residual) | reinterpret_cast<uintptr_t>(weight) | reinterpret_cast<uintptr_t>(x_out)) & 15)
    return fail(SSM_ERR_ARG, "pointers must be 16-B aligned");
  tp->launches++;
  CU(launch_rmsnorm(tp->bf16, residual, weight, eps, x_out, M, tp->cfg.d_model, reinterpret_cast<cudaStream_t>(stream)));
  return SSM_OK;
}

ssm_status_t ssm_tp_check(ssm_tp_t tp, void* stream) {
  if (!tp) return fail(SSM_ERR_ARG, "tp is NULL");
  CU(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  if (tp->k > 1) {
    uint32_t errw = 0;
    CU(cudaMemcpy(&errw, reinterpret_cast<char*>(tp->peers.p[tp->rank]) + 64, 4, cudaMemcpyDeviceToHost));
    if (errw) return fail(SSM_ERR_PROTOCOL, "peer flag wait timed out on rank %d (epoch %u)", tp->rank, tp->epoch);
  }
  return SSM_OK;
}

ssm_status_t ssm_tp_stats(ssm_tp_t tp, int64_t* allreduce_count, int64_t* bytes_sent) {
  if (!tp) return fail(SSM_ERR_ARG, "tp is NULL");
  if (allreduce_count) *allreduce_count = tp->ar_count;
  if (bytes_sent) *bytes_sent = tp->bytes_sent;
  return SSM_OK;
}

ssm_status_t ssm_tp_fused_calls(ssm_tp_t tp, int64_t* calls) {
  if (!tp || !calls) return fail(SSM_ERR_ARG, "NULL argument");
  *calls = tp->fused_calls;
  return SSM_OK;
}

ssm_status_t ssm_tp_epoch(ssm_tp_t tp, uint32_t* epoch) {
  if (!tp || !epoch) return fail(SSM_ERR_ARG, "NULL argument");
  *epoch = tp->epoch;
  return SSM_OK;
}

ssm_status_t ssm_tp_barrier(ssm_tp_t tp, void* stream) {
  if (!tp) return fail(SSM_ERR_ARG, "tp is NULL");
  if (tp->k == 1) return SSM_OK;
  ++tp->epoch;
  tp->launches++;
  PdlScope pdl(!(tp->flags & SSM_COMM_VIRTUAL));
  CU(launch_peer_barrier(tp->peers, tp->rank, tp->k, reinterpret_cast<cudaStream_t>(stream)));
  return SSM_OK;
}

ssm_status_t ssm_tp_launch_count(ssm_tp_t tp, int64_t* launches) {
  if (!tp || !launches) return fail(SSM_ERR_ARG, "NULL argument");
  *launches = tp->launches;
  return SSM_OK;
}

ssm_status_t ssm_dbg_set_gemm_pair(int32_t mode) {
  if (mode < -1 || mode > 1) return fail(SSM_ERR_ARG, "mode=%d (expected -1, 0 or 1)", mode);
  ssm::t_gemm_pair = mode;
  return SSM_OK;
}

ssm_status_t ssm_dbg_gemm(ssm_tp_t tp, const void* A, const void* B, float* C, int32_t M, int32_t N, int32_t K,
                          int32_t swap_ab, int32_t ksplit, void* stream) {
  return ssm_dbg_gemm_ld(tp, A, K, B, K, C, M, N, K, swap_ab, ksplit, stream);
}

ssm_status_t ssm_dbg_gemm_ld(ssm_tp_t tp, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int32_t M,
                             int32_t N, int32_t K, int32_t swap_ab, int32_t ksplit, void* stream) {
  if (!tp || !A || !B || !C) return fail(SSM_ERR_ARG, "NULL argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (ksplit != 1) CU(cudaMemsetAsync(C, 0, (size_t)M * N * 4, s));
  const int kind = ksplit != 1 ? EPI_ATOMIC_F32 : EPI_STORE_F32;
  if (swap_ab)
    CU(gemm(tp, B, ldb, A, lda, N, M, K, ksplit, epi(kind, 1, C, N), s, true));
  else
    CU(gemm(tp, A, lda, B, ldb, M, N, K, ksplit, epi(kind, 0, C, N), s));
  return SSM_OK;
}

ssm_status_t ssm_packed_weight_bytes(int32_t rows, int32_t cols, size_t* bytes) {
  if (!bytes) return fail(SSM_ERR_ARG, "bytes is NULL");
  if (rows <= 0 || cols <= 0) return fail(SSM_ERR_DIM, "rows=%d cols=%d", rows, cols);
  *bytes = packed_blocked_bytes(rows, cols);
  return SSM_OK;
}

ssm_status_t ssm_pack_weight(ssm_tp_t tp, const void* w, int32_t rows, int32_t cols, void* out, size_t out_bytes,
                             void* stream) {
  if (!tp || !w || !out) return fail(SSM_ERR_ARG, "NULL argument");
  if (!tp->bf16) return fail(SSM_ERR_UNSUPPORTED, "packed weights are for the bf16 tensor-core path");
  if (rows <= 0 || cols <= 0) return fail(SSM_ERR_DIM, "rows=%d cols=%d", rows, cols);
  if (out_bytes < packed_blocked_bytes(rows, cols)) return fail(SSM_ERR_ARG, "out buffer too small");
  if ((reinterpret_cast<uintptr_t>(out) & 127) || (reinterpret_cast<uintptr_t>(w) & 15))
    return fail(SSM_ERR_ARG, "w must be 16-B and out 128-B aligned");
  tp->launches++;
  CU(pack_blocked(reinterpret_cast<const __nv_bfloat16*>(w), rows, cols, cols, reinterpret_cast<__nv_bfloat16*>(out),
                  reinterpret_cast<cudaStream_t>(stream)));
  return SSM_OK;
}

ssm_status_t ssm_dbg_gemm_packed(ssm_tp_t tp, const void* X, const void* W, const void* Wpk, float* C, int32_t M,
                                 int32_t N, int32_t K, int32_t ksplit, void* stream) {
  if (!tp || !X || !W || !Wpk || !C) return fail(SSM_ERR_ARG, "NULL argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (ksplit != 1) CU(cudaMemsetAsync(C, 0, (size_t)M * N * 4, s));
  const int kind = ksplit != 1 ? EPI_ATOMIC_F32 : EPI_STORE_F32;
  CU(gemm(tp, W, K, X, K, N, M, K, ksplit, epi(kind, 1, C, N), s, true, Wpk));
  return SSM_OK;
}

ssm_status_t ssm_dbg_scan(ssm_tp_t tp, const void* u, const void* delta, const void* z, int32_t ldz, const float* BC,
                          const float* a_log, const float* d_skip, float* h, void* g, int32_t batch, int32_t seqlen,
                          void* stream) {
  if (!tp || !u || !delta || !z || !BC || !a_log || !d_skip || !h || !g) return fail(SSM_ERR_ARG, "NULL argument");
  const int Ek = tp->Ek, N = tp->cfg.d_state;
  tp->launches++;
  CU(launch_scan(tp->bf16, tp->bf16, u, Ek, delta, Ek, z, ldz, BC, 2 * N, a_log, d_skip, h, (int64_t)Ek * N, g, Ek,
                 batch, seqlen, Ek, N, reinterpret_cast<cudaStream_t>(stream)));
  return SSM_OK;
}

ssm_status_t ssm_rmsnorm_add(ssm_tp_t tp, const float* a, const float* b, const float* weight, float eps, void* x_out,
                             int64_t M, void* stream) {
  if (!tp || !a || !x_out) return fail(SSM_ERR_ARG, "NULL argument");
  if (!tp->bf16) return fail(SSM_ERR_UNSUPPORTED, "ssm_rmsnorm_add: bf16 handles only");
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(weight) |
       reinterpret_cast<uintptr_t>(x_out)) & 15)
    return fail(SSM_ERR_ARG, "pointers must be 16-B aligned");
  PdlScope pdl(M <= 256 && !(tp->flags & SSM_COMM_VIRTUAL));
  tp->launches++;
  CU(launch_rmsnorm2(a, b, 1, weight, eps, reinterpret_cast<__nv_bfloat16*>(x_out), M, tp->cfg.d_model,
                     reinterpret_cast<cudaStream_t>(stream)));
  return SSM_OK;
}

}  // extern "C"

namespace {
struct AttnDims {
  int D, H, hk, d, I, ik;
};
ssm_status_t attn_dims(const ssm_tp_s* t, const ssm_attn_config_t* a, AttnDims* o) {
  if (!a) return fail(SSM_ERR_ARG, "attention config is NULL");
  if (!t->bf16) return fail(SSM_ERR_UNSUPPORTED, "shared attention block: bf16 handles only");
  const int D = t->cfg.d_model, H = a->n_heads, I = a->intermediate;
  if (H < 1 || (2 * D) % H || H % t->k || I < 1 || I % (8 * t->k) || a->max_seq < 1)
    return fail(SSM_ERR_SHARD, "n_heads=%d / intermediate=%d do not split over tp_size=%d (2 d_model=%d)", H, I, t->k,
                2 * D);
  const int d = 2 * D / H;
  if (!(d == 32 || d == 64 || d == 128 || d == 464) || D % 8)
    return fail(SSM_ERR_UNSUPPORTED, "head_dim=%d (supported: 32, 64, 128, 464)", d);
  *o = AttnDims{D, H, H / t->k, d, I, I / t->k};
  return SSM_OK;
}
struct AttnWs {
  size_t xa, qkv, o, a, y, gu, m, dd, mb, part, total;
};
AttnWs attn_ws(const AttnDims& z, int64_t M, int batch = 0, int max_seq = 0) {
  AttnWs L{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += al256(bytes); return o; };
  L.xa = take(M * 2 * z.D * 2);
  L.qkv = take(M * 3 * z.hk * z.d * 2);
  L.o = take(M * z.hk * z.d * 2);
  L.a = take(M * z.D * 4);
  L.y = take(M * z.D * 2);
  L.gu = take(M * 2 * z.ik * 2);
  L.m = take(M * z.ik * 2);
  L.dd = take(M * z.D * 4);
  L.mb = take(M * z.D * 2);
  // decode (one token per sequence): the split-K attention's partials
  L.part = take(batch > 0 && M == batch ? attn_dec_part_floats(batch, z.hk, z.d, max_seq) * 4 : 0);
  L.total = off;
  return L;
}
uint32_t attn_ar_flags(uint32_t flags) {
  if (flags & SSM_AR2_INT8) return 0;
  if (flags & SSM_AR2_FP16) return SSM_QAR_FP16;
  if (flags & SSM_AR2_BF16) return SSM_QAR_BF16;
  return SSM_QAR_FP32;
}
}  // namespace

extern "C" {

ssm_status_t ssm_kv_bytes(ssm_tp_t tp, const ssm_attn_config_t* acfg, int32_t batch, size_t* bytes) {
  if (!tp || !bytes) return fail(SSM_ERR_ARG, "NULL argument");
  AttnDims z;
  ssm_status_t st = attn_dims(tp, acfg, &z);
  if (st != SSM_OK) return st;
  if (batch < 1) return fail(SSM_ERR_DIM, "batch=%d", batch);
  *bytes = 256 + 2 * al256((size_t)batch * acfg->max_seq * z.hk * z.d * 2);
  return SSM_OK;
}

ssm_status_t ssm_kv_alloc(ssm_tp_t tp, const ssm_attn_config_t* acfg, int32_t batch, void* buf, size_t bytes,
                          void* stream, ssm_kv_t* out) {
  if (!out) return fail(SSM_ERR_ARG, "out is NULL");
  *out = nullptr;
  size_t need = 0;
  ssm_status_t st = ssm_kv_bytes(tp, acfg, batch, &need);
  if (st != SSM_OK) return st;
  if (!buf || bytes < need) return fail(SSM_ERR_ARG, "KV buffer NULL or too small (%zu < %zu B)", bytes, need);
  if (reinterpret_cast<uintptr_t>(buf) & 255) return fail(SSM_ERR_ARG, "KV buffer must be 256-B aligned");
  ssm_kv_s* kv = new (std::nothrow) ssm_kv_s();
  if (!kv) return fail(SSM_ERR_ARG, "out of host memory");
  AttnDims z;
  attn_dims(tp, acfg, &z);
  *kv = ssm_kv_s{tp, batch, acfg->max_seq, z.hk, z.d, reinterpret_cast<char*>(buf)};
  if (cudaMemsetAsync(buf, 0, need, reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess) {
    delete kv;
    return fail(SSM_ERR_CUDA, "zero-fill of the KV cache failed");
  }
  *out = kv;
  return SSM_OK;
}

ssm_status_t ssm_kv_reset(ssm_kv_t kv, void* stream) {
  if (!kv) return fail(SSM_ERR_ARG, "kv is NULL");
  CU(cudaMemsetAsync(kv->buf, 0, 256, reinterpret_cast<cudaStream_t>(stream)));   // length and error word
  return SSM_OK;
}

ssm_status_t ssm_kv_free(ssm_kv_t kv) {
  delete kv;
  return SSM_OK;
}

ssm_status_t ssm_attn_workspace_bytes(ssm_tp_t tp, const ssm_attn_config_t* acfg, int32_t batch, int32_t seqlen,
                                      size_t* bytes) {
  if (!tp || !bytes) return fail(SSM_ERR_ARG, "NULL argument");
  AttnDims z;
  ssm_status_t st = attn_dims(tp, acfg, &z);
  if (st != SSM_OK) return st;
  if (batch < 0 || seqlen < 0) return fail(SSM_ERR_DIM, "negative batch/seqlen");
  *bytes = attn_ws(z, (int64_t)batch * seqlen, batch, acfg->max_seq).total;
  return SSM_OK;
}

ssm_status_t ssm_attn_block(ssm_tp_t tp, const ssm_attn_config_t* acfg, const ssm_attn_weights_t* w, ssm_kv_t kv,
                            const float* h, const float* h0, float* t_out, int32_t batch, int32_t seqlen,
                            uint32_t flags, void* workspace, size_t ws_bytes, void* stream) {
  if (!tp) return fail(SSM_ERR_ARG, "tp is NULL");
  AttnDims z;
  ssm_status_t st = attn_dims(tp, acfg, &z);
  if (st != SSM_OK) return st;
  if (!w || !w->norm1 || !w->w_qkv || !w->w_o || !w->norm2 || !w->w_gu || !w->w_d || !w->w_lin)
    return fail(SSM_ERR_ARG, "attention weights struct or one of its pointers is NULL");
  if (!kv || kv->owner != tp) return fail(SSM_ERR_CACHE, "KV cache missing or bound to another handle");
  if (kv->batch != batch || kv->max_seq != acfg->max_seq) return fail(SSM_ERR_CACHE, "KV cache batch/max_seq mismatch");
  if (batch < 0 || seqlen < 0) return fail(SSM_ERR_DIM, "negative batch/seqlen");
  if (!h || !h0 || !t_out) return fail(SSM_ERR_ARG, "h/h0/t_out is NULL");
  if ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(h0) | reinterpret_cast<uintptr_t>(t_out)) & 15)
    return fail(SSM_ERR_ARG, "h/h0/t_out must be 16-B aligned");
  if (flags & ~(uint32_t)(SSM_AR2_INT8 | SSM_AR2_FP16 | SSM_AR2_BF16 | SSM_AR2_FP32))
    return fail(SSM_ERR_ARG, "unknown flags 0x%x", flags);
  const int64_t M = (int64_t)batch * seqlen;
  if (M == 0) return SSM_OK;
  const AttnWs L = attn_ws(z, M, batch, acfg->max_seq);
  if (!workspace || ws_bytes < L.total) return fail(SSM_ERR_ARG, "workspace %zu B < required %zu B", ws_bytes, L.total);
  if (reinterpret_cast<uintptr_t>(workspace) & 255) return fail(SSM_ERR_ARG, "workspace must be 256-B aligned");
  if (tp->k > 1 && (size_t)M * z.D * 4 > half_bytes(tp))
    return fail(SSM_ERR_ARG, "symmetric buffer too small for %lld tokens", (long long)M);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PdlScope pdl(M <= 256 && !(tp->flags & SSM_COMM_VIRTUAL));
  char* W = reinterpret_cast<char*>(workspace);
  auto bf = [&](size_t off) { return reinterpret_cast<__nv_bfloat16*>(W + off); };
  const int D = z.D, A2 = 2 * D, QW = z.hk * z.d;
  int* len = reinterpret_cast<int*>(kv->buf);
  int* err = len + 1;
  __nv_bfloat16* Kc = reinterpret_cast<__nv_bfloat16*>(kv->buf + 256);
  __nv_bfloat16* Vc = reinterpret_cast<__nv_bfloat16*>(kv->buf + 256 + al256((size_t)batch * kv->max_seq * QW * 2));
  // Projections: out[M][N] = X[M][K] W[N][K]^T.  Decode-size calls (M <= 32 tokens) stream the weights
  // through the swap-AB GEMM (weights fill the 128-row MMA tile, the tokens are N; fp32 outputs split
  // over K with atomics into the zeroed output): with the tokens as the 128-row tile a [16 x 3712]
  // output ran on 15 CTAs (0.5 TB/s).
  const bool dec = M <= 32 && tp->bf16;
  auto proj = [&](const void* X, int ldx, const void* Wt, int ldw, int N, int K, int kind, void* out) -> cudaError_t {
    if (!dec) return gemm(tp, X, ldx, Wt, ldw, (int)M, N, K, 1, epi(kind, 0, out, N), s);
    if (kind == EPI_STORE_F32) {
      tp->launches++;
      cudaError_t e = cudaMemsetAsync(out, 0, (size_t)M * N * 4, s);
      if (e != cudaSuccess) return e;
      return gemm(tp, Wt, ldw, X, ldx, N, (int)M, K, split_for(tp, N, K), epi(EPI_ATOMIC_F32, 1, out, N), s, true);
    }
    return gemm(tp, Wt, ldw, X, ldx, N, (int)M, K, 1, epi(kind, 1, out, N), s, true);
  };
  // x = RMSNorm_1(concat(h, h0)); q | k | v of the owned heads
  tp->launches++;
  CU(launch_rmsnorm2(h, h0, 0, w->norm1, acfg->eps, bf(L.xa), M, D, s));
  CU(proj(bf(L.xa), A2, w->w_qkv, A2, 3 * QW, A2, EPI_STORE_BF16, bf(L.qkv)));
  // K, V appended to the cache; causal attention over it; the cache length advanced
  tp->launches += 3;
  CU(launch_kv_append(bf(L.qkv), len, batch, seqlen, z.hk, z.d, kv->max_seq, Kc, Vc, err, s));
  // (the attention reads *len after the append: it counts this call's rows once advanced, so
  //  advance first and let the kernel take t0 = len - L)
  CU(launch_kv_advance(len, seqlen, kv->max_seq, s));
  const float ascale = 1.0f / sqrtf((float)z.d / 2.0f);
  if (seqlen == 1) {  // decode: memory-bound split-K over the cached keys
    tp->launches++;
    CU(launch_attn_decode(bf(L.qkv), len, Kc, Vc, batch, z.hk, z.d, kv->max_seq, ascale,
                          reinterpret_cast<float*>(W + L.part), bf(L.o), s));
  } else {
    CU(launch_attn(bf(L.qkv), len, Kc, Vc, batch, seqlen, z.hk, z.d, kv->max_seq, ascale, bf(L.o), s));
  }
  // a = o W_o^T (row-parallel partial), all-reduced at TP > 1
  float* a = reinterpret_cast<float*>(W + L.a);
  CU(proj(bf(L.o), QW, w->w_o, QW, D, QW, EPI_STORE_F32, a));
  if (tp->k > 1) {
    ssm_status_t r = ssm_qallreduce(tp, a, a, (size_t)M * D, attn_ar_flags(flags), stream);
    if (r != SSM_OK) return r;
  }
  // y = RMSNorm_2(a); m = GELU(y W_g^T) * (y W_u^T); d = m W_d^T (partial), all-reduced
  tp->launches += 2;
  CU(launch_rmsnorm2(a, nullptr, 1, w->norm2, acfg->eps, bf(L.y), M, D, s));
  CU(proj(bf(L.y), D, w->w_gu, D, 2 * z.ik, D, EPI_STORE_BF16, bf(L.gu)));
  CU(launch_gelu_mul(bf(L.gu), M, z.ik, bf(L.m), s));
  float* dd = reinterpret_cast<float*>(W + L.dd);
  CU(proj(bf(L.m), z.ik, w->w_d, z.ik, D, z.ik, EPI_STORE_F32, dd));
  if (tp->k > 1) {
    ssm_status_t r = ssm_qallreduce(tp, dd, dd, (size_t)M * D, attn_ar_flags(flags), stream);
    if (r != SSM_OK) return r;
  }
  // t = m W_lin^T (replicated)
  tp->launches++;
  CU(launch_cast_bf16(dd, M * D, bf(L.mb), s));
  CU(proj(bf(L.mb), D, w->w_lin, D, D, D, EPI_STORE_F32, t_out));
  return SSM_OK;
}

}  // extern "C"

namespace {
struct M2Dims {
  int D, E, Ek, N, P, G, GN, H, Hk, K, Ck, Wp, ldp;
};
ssm_status_t m2_dims(const ssm_tp_s* t, const ssm_m2_config_t* c, M2Dims* o) {
  if (!c) return fail(SSM_ERR_ARG, "Mamba-2 config is NULL");
  if (!t->bf16) return fail(SSM_ERR_UNSUPPORTED, "Mamba-2 mixer: bf16 handles only");
  if (c->headdim != 64 || !(c->d_state == 16 || c->d_state == 64 || c->d_state == 128) || c->n_groups != 1 ||
      c->d_conv < 2 || c->d_conv > 4)
    return fail(SSM_ERR_UNSUPPORTED, "Mamba-2: headdim 64, d_state 16/64/128, n_groups 1, 2 <= d_conv <= 4");
  if (c->d_inner % c->headdim || (c->d_inner / c->headdim) % t->k)
    return fail(SSM_ERR_SHARD, "Mamba-2: heads (%d) do not split over tp_size=%d", c->d_inner / c->headdim, t->k);
  M2Dims z{};
  z.D = t->cfg.d_model;
  z.E = c->d_inner;
  z.Ek = z.E / t->k;
  z.N = c->d_state;
  z.P = c->headdim;
  z.G = c->n_groups;
  z.GN = z.G * z.N;
  z.H = z.E / z.P;
  z.Hk = z.H / t->k;
  z.K = c->d_conv;
  z.Ck = z.Ek + 2 * z.GN;
  z.Wp = 2 * z.Ek + 2 * z.GN + z.Hk;
  z.ldp = (z.Wp + 7) / 8 * 8;  // 16-B rows for the conv kernels' vector loads
  *o = z;
  return SSM_OK;
}
struct M2Ws {
  size_t proj, u, ss, o, part, total;
};
M2Ws m2_ws(const ssm_tp_s* t, const M2Dims& z, int64_t M) {
  M2Ws L{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += al256(bytes); return o; };
  L.proj = take(M * z.ldp * 2);
  L.u = take(M * z.Ck * 2);
  L.ss = take(((M + 3) / 4 * 4) * 4);
  L.o = take(M * z.Ek * 2);
  L.part = take(t->k > 1 ? M * z.D * 4 : 0);
  L.total = off;
  return L;
}
}  // namespace

extern "C" {

ssm_status_t ssm_m2_state_bytes(ssm_tp_t tp, const ssm_m2_config_t* cfg, int32_t batch, size_t* conv_bytes,
                                size_t* h_bytes) {
  if (!tp || !conv_bytes || !h_bytes) return fail(SSM_ERR_ARG, "NULL argument");
  M2Dims z;
  ssm_status_t st = m2_dims(tp, cfg, &z);
  if (st != SSM_OK) return st;
  if (batch < 1) return fail(SSM_ERR_DIM, "batch=%d", batch);
  *conv_bytes = (size_t)batch * (z.K - 1) * z.Ck * 2;
  *h_bytes = (size_t)batch * z.Hk * z.P * z.N * 4;
  return SSM_OK;
}

ssm_status_t ssm_m2_workspace_bytes(ssm_tp_t tp, const ssm_m2_config_t* cfg, int32_t batch, int32_t seqlen,
                                    size_t* bytes) {
  if (!tp || !bytes) return fail(SSM_ERR_ARG, "NULL argument");
  M2Dims z;
  ssm_status_t st = m2_dims(tp, cfg, &z);
  if (st != SSM_OK) return st;
  if (batch < 0 || seqlen < 0) return fail(SSM_ERR_DIM, "negative batch/seqlen");
  *bytes = m2_ws(tp, z, (int64_t)batch * seqlen).total;
  return SSM_OK;
}

ssm_status_t ssm_m2_mixer(ssm_tp_t tp, const ssm_m2_config_t* cfg, const ssm_m2_weights_t* w, void* conv_state,
                          float* h_state, const void* x_in, float* residual, int32_t batch, int32_t seqlen,
                          uint32_t flags, void* workspace, size_t ws_bytes, void* stream) {
  if (!tp) return fail(SSM_ERR_ARG, "tp is NULL");
  M2Dims z;
  ssm_status_t st = m2_dims(tp, cfg, &z);
  if (st != SSM_OK) return st;
  if (!w || !w->w_in || !w->conv_w || !w->conv_b || !w->dt_bias || !w->a_log || !w->d_skip || !w->norm_w || !w->w_out)
    return fail(SSM_ERR_ARG, "Mamba-2 weights struct or one of its pointers is NULL");
  if (!conv_state || !h_state || !x_in || !residual) return fail(SSM_ERR_ARG, "NULL state / input / residual");
  if ((reinterpret_cast<uintptr_t>(conv_state) | reinterpret_cast<uintptr_t>(h_state) |
       reinterpret_cast<uintptr_t>(x_in) | reinterpret_cast<uintptr_t>(residual)) & 15)
    return fail(SSM_ERR_ARG, "pointers must be 16-B aligned");
  if (batch < 0 || seqlen < 0) return fail(SSM_ERR_DIM, "negative batch/seqlen");
  if (flags & ~(uint32_t)(SSM_AR2_INT8 | SSM_AR2_FP32 | SSM_AR2_FP16 | SSM_AR2_BF16))
    return fail(SSM_ERR_ARG, "unknown flags 0x%x", flags);
  const int64_t M = (int64_t)batch * seqlen;
  if (M == 0) return SSM_OK;
  const M2Ws L = m2_ws(tp, z, M);
  if (!workspace || ws_bytes < L.total) return fail(SSM_ERR_ARG, "workspace %zu B < required %zu B", ws_bytes, L.total);
  if (reinterpret_cast<uintptr_t>(workspace) & 255) return fail(SSM_ERR_ARG, "workspace must be 256-B aligned");
  if (tp->k > 1 && (size_t)M * z.D * 4 > half_bytes(tp))
    return fail(SSM_ERR_ARG, "symmetric buffer too small for %lld tokens", (long long)M);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PdlScope pdl(seqlen == 1 && M <= 256 && !(tp->flags & SSM_COMM_VIRTUAL));
  char* W = reinterpret_cast<char*>(workspace);
  __nv_bfloat16* proj = reinterpret_cast<__nv_bfloat16*>(W + L.proj);
  __nv_bfloat16* u = reinterpret_cast<__nv_bfloat16*>(W + L.u);
  float* ss = reinterpret_cast<float*>(W + L.ss);
  __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(W + L.o);
  // packed in_proj [z | x | B | C | dt] of the rank (decode: swap-AB, the weights fill the MMA rows)
  const bool swap = seqlen == 1 && batch <= 32;
  // (its epilogue also zeroes ss, which the scan accumulates the gated rows' sums of squares into)
  {
    Epilogue e = epi(EPI_STORE_BF16, swap ? 1 : 0, proj, z.ldp);
    e.zero = ss;
    e.nzero = (M + 3) / 4 * 4;
    if (swap)
      CU(gemm(tp, w->w_in, z.D, x_in, z.D, z.Wp, (int)M, z.D, 1, e, s, true));
    else
      CU(gemm(tp, x_in, z.D, w->w_in, z.D, (int)M, z.Wp, z.D, 1, e, s));
  }
  // causal conv + SiLU over the x | B | C channels (window of the cache updated)
  const __nv_bfloat16* xbc = proj + z.Ek;
  if (seqlen == 1) {
    tp->launches++;
    CU(launch_conv_decode(1, xbc, z.ldp, conv_state, w->conv_w, w->conv_b, u, z.Ck, batch, z.Ck, z.K, nullptr, 0,
                          nullptr, 0, nullptr, s));
  } else {
    tp->launches += 2;
    CU(launch_conv1d_silu(1, xbc, z.ldp, conv_state, w->conv_w, w->conv_b, u, z.Ck, batch, seqlen, z.Ck, z.K, s));
    CU(launch_conv_state_update(1, xbc, z.ldp, conv_state, batch, seqlen, z.Ck, z.K, s));
  }
  // scan (per head, per sequence) with the gate, the norm weight and the rows' sums of squares
  // fused into its output (o = bf16(y SiLU(z) w)); (TP > 1) all-reduce of the sums; the out_proj
  // epilogues scale each row by 1 / sqrt(ss / E + eps) (reading M3)
  tp->launches += 1;
  CU(launch_m2_scan(proj, z.ldp, 2 * z.Ek + 2 * z.GN, u, z.Ck, z.Ek, z.Ek + z.GN, z.H / z.G / tp->k > 0 ? z.Hk : 1,
                    w->dt_bias, w->a_log, w->d_skip, w->norm_w, h_state, o, z.Ek, ss, batch, seqlen, z.Hk, z.P, z.N,
                    s));
  if (tp->k > 1) {
    ssm_status_t r = ssm_qallreduce(tp, ss, ss, (size_t)((M + 3) / 4 * 4), SSM_QAR_FP32, stream);
    if (r != SSM_OK) return r;
  }
  auto oepi = [&](int kind, int trans, float* C) {
    Epilogue e = epi(kind, trans, C, z.D);
    e.rss = ss;
    e.rss_inv = 1.0f / (float)z.E;
    e.rss_eps = cfg->eps;
    return e;
  };
  // out_proj (row-parallel): TP = 1 straight into the residual, else partial + AR#2 (decode:
  // swap-AB split-K with fp32 atomics)
  if (tp->k == 1) {
    if (swap)
      CU(gemm(tp, w->w_out, z.Ek, o, z.Ek, z.D, (int)M, z.Ek, split_for(tp, z.D, z.Ek),
              oepi(EPI_ATOMIC_F32, 1, residual), s, true));
    else
      CU(gemm(tp, o, z.Ek, w->w_out, z.Ek, (int)M, z.D, z.Ek, 1, oepi(EPI_ADD_F32, 0, residual), s));
  } else {
    float* part = reinterpret_cast<float*>(W + L.part);
    if (swap) {
      CU(cudaMemsetAsync(part, 0, (size_t)M * z.D * 4, s));
      CU(gemm(tp, w->w_out, z.Ek, o, z.Ek, z.D, (int)M, z.Ek, split_for(tp, z.D, z.Ek),
              oepi(EPI_ATOMIC_F32, 1, part), s, true));
    } else {
      CU(gemm(tp, o, z.Ek, w->w_out, z.Ek, (int)M, z.D, z.Ek, 1, oepi(EPI_STORE_F32, 0, part), s));
    }
    const uint32_t qf = (flags & SSM_AR2_FP32) ? SSM_QAR_FP32 : (flags & SSM_AR2_FP16) ? SSM_QAR_FP16
                      : (flags & SSM_AR2_BF16) ? SSM_QAR_BF16 : 0;
    ssm_status_t r = ssm_qallreduce(tp, part, residual, (size_t)M * z.D, qf | SSM_QAR_ACCUMULATE, stream);
    if (r != SSM_OK) return r;
  }
  return SSM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- persistent whole-stack decode
struct ssm_dstack_s {
  ssm_tp_s* owner;
  int L, batch, ctas;
  float eps;
  DsGeom g;
  std::vector<DsLayer> table;  // host copy of the device layer table (source of the async upload)
  DsLayer* table_dev;
  uint8_t* scratch;
  unsigned long long* trace = nullptr;  // ssm_dbg_dstack_trace
};

namespace {
size_t al256z(size_t x) { return (x + 255) & ~size_t(255); }

ssm_status_t dstack_geom(ssm_tp_s* t, int32_t n_layers, int32_t batch, int32_t ctas, DsGeom* g, size_t* bytes) {
  if (!t) return fail(SSM_ERR_ARG, "tp is NULL");
  const ssm_config_t& c = t->cfg;
  if (t->k != 1 || !t->bf16 || c.n_heads != 1 || c.d_state != 16)
    return fail(SSM_ERR_UNSUPPORTED, "persistent decode: tp_size 1, bf16, n_heads 1, d_state 16 only");
  if (n_layers < 1 || batch < 1 || batch > 16) return fail(SSM_ERR_UNSUPPORTED, "persistent decode: n_layers >= 1, batch 1..16");
  const int nc = ctas > 0 ? ctas : t->num_sms;
  if (nc > t->num_sms) return fail(SSM_ERR_ARG, "ctas=%d > %d SMs (one CTA per SM)", nc, t->num_sms);
  *g = ds_geometry(batch, c.d_model, c.d_inner, c.dt_rank, t->P, c.d_conv, nc);
  if (!g->ok)
    return fail(SSM_ERR_UNSUPPORTED, "persistent decode: shape not supported (d_model=%d d_inner=%d dt_rank=%d batch=%d ctas=%d)",
                c.d_model, c.d_inner, c.dt_rank, batch, nc);
  *bytes = al256z((size_t)n_layers * ds_packed_layer_bytes(c.d_model, c.d_inner, c.dt_rank, t->P)) +
           al256z((size_t)n_layers * sizeof(DsLayer)) + al256z(g->scratch_bytes);
  return SSM_OK;
}
}  // namespace

extern "C" {

ssm_status_t ssm_dstack_bytes(ssm_tp_t tp, int32_t n_layers, int32_t batch, int32_t ctas, size_t* bytes) {
  if (!bytes) return fail(SSM_ERR_ARG, "bytes is NULL");
  DsGeom g;
  return dstack_geom(tp, n_layers, batch, ctas, &g, bytes);
}

ssm_status_t ssm_dstack_create(ssm_tp_t tp, int32_t n_layers, const ssm_layer_weights_t* layers,
                               const ssm_state_t* states, int32_t batch, float norm_eps, int32_t ctas, void* buf,
                               size_t buf_bytes, void* stream, ssm_dstack_t* out) {
  if (!out) return fail(SSM_ERR_ARG, "out is NULL");
  *out = nullptr;
  DsGeom g;
  size_t need = 0;
  ssm_status_t st = dstack_geom(tp, n_layers, batch, ctas, &g, &need);
  if (st != SSM_OK) return st;
  if (!layers || !states) return fail(SSM_ERR_ARG, "layers/states is NULL");
  if (!buf || buf_bytes < need) return fail(SSM_ERR_ARG, "buffer %zu B < required %zu B", buf_bytes, need);
  if (reinterpret_cast<uintptr_t>(buf) & 255) return fail(SSM_ERR_ARG, "buffer must be 256-B aligned");
  const int nc = ctas > 0 ? ctas : tp->num_sms;
  if (ds_max_active(g.smem) < 1) return fail(SSM_ERR_CUDA, "persistent decode kernel cannot be resident (%d B smem)", g.smem);
  const ssm_config_t& c = tp->cfg;
  const int D = c.d_model, E = c.d_inner, R = c.dt_rank, P = tp->P;
  for (int l = 0; l < n_layers; ++l) {
    const ssm_layer_weights_t& w = layers[l];
    if (!w.w_in || !w.w_out || !w.w_x || !w.w_dt || !w.conv_w || !w.conv_b || !w.b_dt || !w.a_log || !w.d_skip)
      return fail(SSM_ERR_ARG, "layer %d: a weight pointer is NULL", l);
    if (!states[l] || states[l]->owner != tp || states[l]->batch != batch)
      return fail(SSM_ERR_CACHE, "layer %d: state missing, of another handle or of another batch", l);
  }
  ssm_dstack_s* ds = new (std::nothrow) ssm_dstack_s();
  if (!ds) return fail(SSM_ERR_ARG, "out of host memory");
  ds->owner = tp;
  ds->L = n_layers;
  ds->batch = batch;
  ds->ctas = nc;
  ds->eps = norm_eps;
  ds->g = g;
  ds->table.resize(n_layers);
  uint8_t* p = reinterpret_cast<uint8_t*>(buf);
  const size_t lb = ds_packed_layer_bytes(D, E, R, P);
  uint8_t* packed = p;
  ds->table_dev = reinterpret_cast<DsLayer*>(p + al256z((size_t)n_layers * lb));
  ds->scratch = reinterpret_cast<uint8_t*>(ds->table_dev) + al256z((size_t)n_layers * sizeof(DsLayer));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int l = 0; l < n_layers; ++l) {
    const ssm_layer_weights_t& w = layers[l];
    uint8_t* dst = packed + (size_t)l * lb;
    cudaError_t e = ds_pack_layer(reinterpret_cast<const __nv_bfloat16*>(w.w_in), reinterpret_cast<const __nv_bfloat16*>(w.w_out),
                                  reinterpret_cast<const __nv_bfloat16*>(w.w_x), reinterpret_cast<const __nv_bfloat16*>(w.w_dt),
                                  D, E, R, P, dst, s);
    if (e == cudaSuccess)
      e = ds_fill_layer(&ds->table[l], dst, D, E, R, P, w.conv_w, w.conv_b, w.b_dt, w.a_log, w.d_skip, states[l]->conv,
                        states[l]->h);
    if (e != cudaSuccess) {
      delete ds;
      return fail(SSM_ERR_CUDA, "packing layer %d: %s", l, cudaGetErrorString(e));
    }
  }
  if (cudaMemcpyAsync(ds->table_dev, ds->table.data(), (size_t)n_layers * sizeof(DsLayer), cudaMemcpyHostToDevice, s) !=
          cudaSuccess ||
      cudaMemsetAsync(ds->scratch, 0, g.scratch_bytes, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    delete ds;
    return fail(SSM_ERR_CUDA, "uploading the layer table: %s", cudaGetErrorString(cudaGetLastError()));
  }
  *out = ds;
  return SSM_OK;
}

ssm_status_t ssm_dstack_decode(ssm_dstack_t ds, float* residual, void* stream) {
  if (!ds) return fail(SSM_ERR_ARG, "dstack is NULL");
  if (!residual || (reinterpret_cast<uintptr_t>(residual) & 15)) return fail(SSM_ERR_ARG, "residual NULL or not 16-B aligned");
  ssm_tp_s* t = ds->owner;
  const ssm_config_t& c = t->cfg;
  t->launches++;
  CU(ds_launch(ds->table_dev, ds->L, ds->batch, c.d_model, c.d_inner, c.dt_rank, t->P, c.d_conv, ds->eps, c.bcdt_rmsnorm,
               c.rms_eps, residual, ds->scratch, ds->g, ds->ctas, reinterpret_cast<cudaStream_t>(stream), ds->trace));
  return SSM_OK;
}

ssm_status_t ssm_dbg_dstack_trace(ssm_dstack_t ds, void* trace) {
  if (!ds) return fail(SSM_ERR_ARG, "dstack is NULL");
  ds->trace = reinterpret_cast<unsigned long long*>(trace);
  return SSM_OK;
}

ssm_status_t ssm_dstack_destroy(ssm_dstack_t ds) {
  delete ds;
  return SSM_OK;
}

}  // extern "C"
