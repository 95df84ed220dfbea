// decode_stack.cu — persistent whole-stack decode at TP = 1: ONE cooperative launch per token runs
// every layer's pre-norm + mixer decode step (SURVEY.md §8 rows a1-a7 at L = 1, a10, a11;
// PAPER.md:276-287 §4.1 "decode from the cached state", §2.2 the mixer).
//
// Why a persistent kernel: a decode token is a weight stream (W_in 2E x D, W_out D x E, W_x, W_dt:
// ~82 MB per Mamba-2.8B layer at batch 16) plus a latency-bound middle (conv step, x_proj reduction,
// scan step).  The per-layer graph (4 kernels per layer) measured ~34 us per layer against a 14.5 us
// HBM floor: ~10 us of kernel-boundary latency and an in_proj that streams on 80 of 148 SMs.
// Here every SM streams its share of every layer's weights through one shared-memory ring that
// runs ahead across phases and layers (weights never depend on activations), and the three
// data-dependent steps are separated by grid barriers instead of kernel boundaries:
//
//   per layer l:
//   A  every CTA reads the fp32 residual into bf16 A fragments and forms the RMSNorm statistic;
//      in_proj units (8 rows x D): xz = rstd[b] * (W_in bf16(r));  x rows -> conv step + SiLU -> u,
//      window shift, x_proj partial (mma m16n8k8) -> red.add into xacc;  z rows -> z      | barrier
//   B  channel groups: dt = softplus(W_dt dt_low + b_dt) (mma m16n8k16), h = exp(dt A) h + dt B u,
//      y = C h + D u, g = y SiLU(z) -> g in A-fragment order; h written back            | barrier
//   C  out_proj units (8 rows x E/4): r += W_out g (red.add)                               | barrier
//
// Pre-norm (reading Q16: RMSNorm, weight 1, eps): the norm is applied after the in_proj contraction,
// xz[b] = rstd[b] * (W_in bf16(r[b])) -- the same product as W_in bf16(rstd[b] r[b]) up to where the
// bf16 rounding of the GEMM input falls (reading Q22).
//
// CTA roles (512 threads, 1 CTA per SM): warps 0-10 "MMA warps" (mma.sync over bf16 fragments
// pre-packed in global memory: weights stream in through the ring and are read with one LDS.128 per
// lane per 32-wide k chunk; activations are register-resident A fragments), warps 11-14 "epilogue
// warps" (cross-warp reduction of a unit's 8 partials, conv step / z store / x_proj / residual
// update), warp 15 the producer (one lane issues cp.async.bulk copies of whole units into the ring).
// Decode GEMMs at batch <= 16 are HBM-bound weight streams (16 flop per weight byte): the tensor
// pipe of mma.sync is far from the bound, what matters is keeping every SM's stream fed.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace ssm {

namespace {

constexpr int kMW = 11;                     // MMA warps
constexpr int kEW = 4;                      // epilogue warps
constexpr int kThreads = (kMW + kEW + 1) * 32;  // + the producer warp: 16 warps, 128 registers per thread
constexpr int kWork = (kMW + kEW) * 32;     // threads in grid barriers and phase B
constexpr int kSlots = 8;                   // ring units in flight (mbarrier slots)
constexpr int kMaxCA = 8;                   // phase A: 32-wide k chunks per MMA warp (D <= 2816)
constexpr int kMaxCC = 4;                   // phase C: chunks per MMA warp per quarter (E <= 5632)
constexpr int kMaxPT = 8;                   // x_proj 8-wide p tiles per epilogue warp (P <= 256)
constexpr int kMaxXU = 5;                   // in_proj x units (8 channels) per CTA
constexpr int kRB = 4;                      // reduction buffers: the MMA warps run up to 3 units ahead
constexpr int kL2AheadIdle = 8;             // ... and while the ring is full (8 / 12 / 16 measured equal)
constexpr int kL2Ahead = 3;                 // ring units prefetched into L2 ahead of the ring

SSM_DEV void mma_1688_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(b0));
}
SSM_DEV uint32_t ld_acquire_gpu_u32(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SSM_DEV uint4 lds128(uint32_t addr) {  // shared-window address: LDS.128, not a generic load
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
SSM_DEV uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}
SSM_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__host__ __device__ inline int part(int n, int c, int nc) { return (n * c) / nc; }  // (n * c < 2^31 here)

}  // namespace

struct DsArgs {
  const DsLayer* layers;
  int L, B, D, E, R, P, K;
  float eps;
  int bcdt_rmsnorm;
  float rms_eps;
  float* r;                 // residual [B][D] fp32, updated in place through all layers
  __nv_bfloat16* g;         // gated output [16][E] (rows >= B stay zero)
  __nv_bfloat16* u;         // [B][E]
  __nv_bfloat16* z;         // [B][E]
  float* xacc;              // [2][16][P]  (zero between uses)
  unsigned* bar;            // [2] grid-barrier counter, exit counter
  int ring_bytes, nch_max;  // ring size; max phase-B channels per CTA
  unsigned long long* trace; // debug (ssm_dbg_dstack_trace): [grid][L][32] globaltimer stamps, or NULL
  int off_sb, off_red, off_pb, off_ut, off_misc;
};

namespace {

// Shared-memory carve-up: everything is an offset from the 1 KB-aligned base, recomputed from the
// (constant-bank) kernel parameters at each use so no pointer stays live in a register.
struct Smem {
  uint8_t* base;
  const DsArgs* a;
  SSM_DEV uint8_t* ring() const { return base; }
  SSM_DEV float* sh() const { return reinterpret_cast<float*>(base + a->off_sb); }                 // [B][nch_max][16]
  SSM_DEV uint32_t* swdt() const { return reinterpret_cast<uint32_t*>(base + a->off_sb + a->B * a->nch_max * 64); }
  SSM_DEV float* salog() const {                                                                    // [nch_max][16]
    return reinterpret_cast<float*>(base + a->off_sb + a->B * a->nch_max * 64 + (a->nch_max / 8) * (a->R / 16) * 256);
  }
  SSM_DEV float* sbdt() const { return salog() + a->nch_max * 16; }
  SSM_DEV float* sdsk() const { return sbdt() + a->nch_max; }
  SSM_DEV float* sred() const { return reinterpret_cast<float*>(base + a->off_red); }              // [kRB][kMW][128]
  SSM_DEV float* sdbc() const { return reinterpret_cast<float*>(base + a->off_pb); }  // [16][P + 8] (bank shift per row)
  SSM_DEV float* sdt() const { return sdbc() + 16 * (a->P + 8); }                                   // [16][nch_max]
  SSM_DEV float* sA() const { return sdt() + 16 * a->nch_max; }                                      // [nch_max][16]
  SSM_DEV __nv_bfloat16* su() const { return reinterpret_cast<__nv_bfloat16*>(sA() + a->nch_max * 16); }  // [16][nch_max]
  SSM_DEV __nv_bfloat16* sz() const { return su() + 16 * a->nch_max; }                                    // [16][nch_max]
  SSM_DEV __nv_bfloat16* utile() const { return reinterpret_cast<__nv_bfloat16*>(base + a->off_ut); }  // [2][16][8]
  SSM_DEV uint64_t* full() const { return reinterpret_cast<uint64_t*>(base + a->off_misc); }     // [kSlots]
  SSM_DEV uint64_t* empty() const { return full() + kSlots; }                                       // [kSlots]
  SSM_DEV uint64_t* ready() const { return full() + 2 * kSlots; }                                   // [kRB]
  SSM_DEV uint64_t* freeb() const { return full() + 2 * kSlots + kRB; }                             // [kRB]
  SSM_DEV uint64_t* mbB() const { return full() + 2 * kSlots + 2 * kRB; }                           // phase-B prefetch
  SSM_DEV uint64_t* mbX() const { return full() + 2 * kSlots + 2 * kRB + 1; }                       // phase-A prefetch
  SSM_DEV uint64_t* mbSS() const { return full() + 2 * kSlots + 2 * kRB + 2; }                      // pre-norm partials
  SSM_DEV float* ssp() const { return reinterpret_cast<float*>(full() + 2 * kSlots + 2 * kRB + 3); }  // [kMW][16]
  SSM_DEV struct Pump* pump() const { return reinterpret_cast<struct Pump*>(base + a->off_misc + 1024); }
  // phase-A epilogue operands of this CTA's x units (aliasing the phase-B scratch, free during C and A):
  // W_x B fragments [kMaxXU][P/8][32] u32, conv taps [kMaxXU * 8][K], conv bias [kMaxXU * 8], windows
  // [kMaxXU][16 b][3 j][8 n] bf16
  SSM_DEV uint32_t* sxw() const { return reinterpret_cast<uint32_t*>(base + a->off_pb); }
  SSM_DEV float* sxcw() const { return reinterpret_cast<float*>(base + a->off_pb + kMaxXU * a->P * 16); }
  SSM_DEV float* sxcb() const { return sxcw() + kMaxXU * 8 * 4; }
  SSM_DEV uint16_t* sxwin() const { return reinterpret_cast<uint16_t*>(sxcb() + kMaxXU * 8); }
};

// Grid barrier over the work threads of every CTA (the producer warp never joins): bar.sync, then one
// thread per CTA releases its arrival and spins on the counter with acquire loads (bar.sync orders
// the CTA's other threads' writes before that release).
SSM_DEV void grid_sync(unsigned* bar, unsigned target) {
  named_bar_sync(1, kWork);
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (ld_acquire_gpu_u32(bar) < target) {
    }
  }
  named_bar_sync(1, kWork);
}

// Phase-B prefetch of layer l (h tile, W_dt fragments, A_log, b_dt, D for this CTA's channels):
// one thread issues bulk copies that complete on mbB.
SSM_DEV void issue_phase_b_prefetch(const DsArgs& a, const Smem& s, const DsLayer& ly, int gb0, int gb1) {
  const int nch = 8 * (gb1 - gb0), d0 = 8 * gb0;
  const uint32_t hb = (uint32_t)nch * 64, wb = (uint32_t)(gb1 - gb0) * (a.R / 16) * 256;
  const uint32_t tot = (uint32_t)a.B * hb + wb + hb + 2u * nch * 4;
  mbar_arrive_expect_tx(s.mbB(), tot);
  if (nch == 0) return;  // (tiny shapes: a CTA without phase-B channels)
  for (int b = 0; b < a.B; ++b)
    bulk_g2s(s.sh() + (size_t)b * a.nch_max * 16, ly.h + ((size_t)b * a.E + d0) * 16, hb, s.mbB());
  bulk_g2s(s.swdt(), ly.wdt + (size_t)gb0 * (a.R / 16) * 256, wb, s.mbB());
  bulk_g2s(s.salog(), ly.a_log + (size_t)d0 * 16, hb, s.mbB());
  bulk_g2s(s.sbdt(), ly.b_dt + d0, nch * 4, s.mbB());
  bulk_g2s(s.sdsk(), ly.d_skip + d0, nch * 4, s.mbB());
}

// Phase-A prefetch of layer l (W_x fragments, conv taps and bias of this CTA's x groups [gx0, gx1)):
// one thread issues bulk copies that complete on mbX.
SSM_DEV void issue_phase_a_prefetch(const DsArgs& a, const Smem& s, const DsLayer& ly, int gx0, int gx1) {
  const int ng = gx1 - gx0;
  const uint32_t wb = (uint32_t)ng * (a.P / 8) * 128, cwb = (uint32_t)ng * 8 * a.K * 4, cbb = (uint32_t)ng * 32;
  mbar_arrive_expect_tx(s.mbX(), wb + cwb + cbb);
  if (ng == 0) return;
  bulk_g2s(s.sxw(), ly.wxf + (size_t)gx0 * (a.P / 8) * 32, wb, s.mbX());
  bulk_g2s(s.sxcw(), ly.conv_w + (size_t)gx0 * 8 * a.K, cwb, s.mbX());
  bulk_g2s(s.sxcb(), ly.conv_b + (size_t)gx0 * 8, cbb, s.mbX());
}

// The cached conv windows of this CTA's x groups (16-B rows of 8 channels per (group, b, tap)) ->
// sxwin by cp.async from the epilogue threads (waited for at the start of the layer's phase A).
SSM_DEV void issue_window_prefetch(const DsArgs& a, const Smem& s, const DsLayer& ly, int gx0, int gx1, int e) {
  const int B = a.B, K = a.K;
  const uint16_t* cst = reinterpret_cast<const uint16_t*>(ly.cst);
  for (int q = e; q < (gx1 - gx0) * B * (K - 1); q += kEW * 32) {
    const int xi = q / (B * (K - 1)), r = q % (B * (K - 1)), bb = r / (K - 1), j = r % (K - 1);
    cp_async16(s.sxwin() + ((xi * 16 + bb) * 3 + j) * 8, cst + ((size_t)bb * (K - 1) + j) * a.E + 8 * (gx0 + xi), true);
  }
  cp_async_commit();
}

// Ring producer state (lane 0 of the producer warp).
struct Pump {
  long long issued, released;
  int seq, oldest, pf, nA, nC, ua0, uc0, szA, szC, total;
};

SSM_DEV int pump_size(const Pump& p, int q) { return q % (p.nA + p.nC) < p.nA ? p.szA : p.szC; }
SSM_DEV const uint8_t* pump_src(const DsArgs& a, const Pump& p, int q) {
  const int l = q / (p.nA + p.nC), pos = q % (p.nA + p.nC);
  const DsLayer& ly = a.layers[l];
  return pos < p.nA ? ly.wa + (size_t)(p.ua0 + pos) * p.szA : ly.wc + (size_t)(p.uc0 + pos - p.nA) * p.szC;
}

// Issue units while the ring has room (waiting for the oldest unit's release when it has none).
__device__ __forceinline__ void pump_run(const DsArgs& a, const Smem& s, Pump* pp) {
  Pump p = *pp;
  while (p.seq < p.total) {
    const int sz = pump_size(p, p.seq);
    while (p.seq - p.oldest >= kSlots || p.issued + sz - p.released > a.ring_bytes) {
      // the ring is full, so the consumers are in a latency-bound step (scan step, barrier, phase start)
      // and HBM is idle: prefetch deeper into L2 while waiting
      while (!mbar_try_wait(&s.empty()[p.oldest % kSlots], (p.oldest / kSlots) & 1))
        if (p.pf < p.total && p.pf < p.seq + 1 + kL2AheadIdle) {
          prefetch_l2(pump_src(a, p, p.pf), (uint32_t)pump_size(p, p.pf));
          ++p.pf;
        }
      p.released += pump_size(p, p.oldest);
      ++p.oldest;
    }
    // L2 prefetch kL2Ahead units beyond the ring: while the ring is full during the latency-bound steps
    // (scan step, barriers, phase starts) HBM keeps streaming the next units into L2 (deeper lookahead
    // measured: 2-3 best; 6 +1.5%, 8 +3%, 16 +12%, 32 +30% per Mamba-2.8B layer)
    for (; p.pf < p.total && p.pf < p.seq + 1 + kL2Ahead; ++p.pf)
      prefetch_l2(pump_src(a, p, p.pf), (uint32_t)pump_size(p, p.pf));
    const uint8_t* src = pump_src(a, p, p.seq);
    const int off = (int)(p.issued % a.ring_bytes);
    uint64_t* fb = &s.full()[p.seq % kSlots];
    mbar_arrive_expect_tx(fb, (uint32_t)sz);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int first = min(sz, a.ring_bytes - off);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(s.ring() + off)),
        "l"(src), "r"(first), "r"(smem_u32(fb)), "l"(pol)
        : "memory");
    if (first < sz)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              smem_u32(s.ring())),
          "l"(src + first), "r"(sz - first), "r"(smem_u32(fb)), "l"(pol)
          : "memory");
    p.issued += sz;
    ++p.seq;
  }
  *pp = p;
}

// Debug timeline: slot k of (CTA, layer) <- globaltimer (one thread per stamp; NULL trace = off).
SSM_DEV void stamp(const DsArgs& a, int l, int k) {
  if (a.trace) a.trace[((size_t)blockIdx.x * a.L + l) * 32 + k] = globaltimer();
}

// Unit-sequence counters shared by the MMA and epilogue warps: ring unit index (mbarrier slot /
// parity), reduction-buffer unit index, ring byte offset of the next unit.
struct Ctr {
  int seq, useq, roff;
};

// The MMA warps' unit loop: weight B fragments from the ring (one LDS.128 per lane per 32-wide chunk),
// activation A fragments in registers, partial [16 x 8] -> the unit's reduction buffer.
template <int MAXC>
SSM_DEV Ctr unit_loop(const DsArgs& a, const Smem& s, const uint32_t (&xa)[MAXC][8], int nch, int u0, int u1, int sz,
                      Ctr ct) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ring = smem_u32(s.ring());
  for (int u = u0; u < u1; ++u, ++ct.seq, ++ct.useq) {
    const int slot = ct.seq % kSlots;
    mbar_wait(&s.full()[slot], (ct.seq / kSlots) & 1);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int j = warp + kMW * i;
      if (j < nch) {
        int o = ct.roff + j * 512 + lane * 16;
        if (o >= a.ring_bytes) o -= a.ring_bytes;
        const uint4 w4 = lds128(ring + o);
        const uint32_t a0[4] = {xa[i][0], xa[i][1], xa[i][2], xa[i][3]};
        const uint32_t a1[4] = {xa[i][4], xa[i][5], xa[i][6], xa[i][7]};
        mma_16816_bf16(acc, a0, w4.x, w4.y);
        mma_16816_bf16(acc, a1, w4.z, w4.w);
      }
    }
    mbar_arrive(&s.empty()[slot]);
    mbar_wait(&s.freeb()[ct.useq % kRB], ((ct.useq / kRB) & 1) ^ 1);
    float* sp = s.sred() + (ct.useq % kRB) * (kMW * 128) + warp * 128;
    sp[lane] = acc[0]; sp[32 + lane] = acc[1]; sp[64 + lane] = acc[2]; sp[96 + lane] = acc[3];
    mbar_arrive(&s.ready()[ct.useq % kRB]);
    ct.roff += sz;
    if (ct.roff >= a.ring_bytes) ct.roff -= a.ring_bytes;
  }
  return ct;
}

// Phase A, MMA warps: A fragments = bf16(r) straight from the fp32 residual (this warp's 32-wide k
// chunks j = warp + kMW i of all 16 rows; rows >= B zero) plus the warp's share of the pre-norm sum
// of squares per token -> ssp[warp][b] (the CTA's warps together cover all of D, so every CTA forms
// the full RMSNorm statistic itself).
__device__ __forceinline__ Ctr mma_units_a(const DsArgs& a, uint8_t* base, int l, int u0, int u1, Ctr ct) {
  const Smem s{base, &a};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b0 = lane >> 2, b1 = b0 + 8, q2 = 2 * (lane & 3);
  const int D = a.D, nch = D / 32;
  const bool v0 = b0 < a.B, v1 = b1 < a.B;
  const float* r0 = a.r + (size_t)b0 * D;
  const float* r1 = a.r + (size_t)b1 * D;
  uint32_t xa[kMaxCA][8];
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxCA; ++i) {
    const int j = min(warp + kMW * i, nch - 1);
    const bool in = warp + kMW * i < nch;
    const int k = 32 * j + 4 * q2;   // this lane's 8 consecutive k of the chunk (permuted fragments)
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 p0 = (in && v0) ? __ldcg(reinterpret_cast<const float4*>(r0 + k)) : z4;
    const float4 p1 = (in && v0) ? __ldcg(reinterpret_cast<const float4*>(r0 + k + 4)) : z4;
    const float4 p2 = (in && v1) ? __ldcg(reinterpret_cast<const float4*>(r1 + k)) : z4;
    const float4 p3 = (in && v1) ? __ldcg(reinterpret_cast<const float4*>(r1 + k + 4)) : z4;
    s0 = fmaf(p0.x, p0.x, fmaf(p0.y, p0.y, fmaf(p0.z, p0.z, fmaf(p0.w, p0.w, s0))));
    s0 = fmaf(p1.x, p1.x, fmaf(p1.y, p1.y, fmaf(p1.z, p1.z, fmaf(p1.w, p1.w, s0))));
    s1 = fmaf(p2.x, p2.x, fmaf(p2.y, p2.y, fmaf(p2.z, p2.z, fmaf(p2.w, p2.w, s1))));
    s1 = fmaf(p3.x, p3.x, fmaf(p3.y, p3.y, fmaf(p3.z, p3.z, fmaf(p3.w, p3.w, s1))));
    // k16 step 0: a0 (row b0, elements 0-1), a1 (row b1, 0-1), a2 (row b0, 2-3), a3 (row b1, 2-3);
    // k16 step 1: the same with elements 4-7
    xa[i][0] = pack_bf2(p0.x, p0.y); xa[i][1] = pack_bf2(p2.x, p2.y);
    xa[i][2] = pack_bf2(p0.z, p0.w); xa[i][3] = pack_bf2(p2.z, p2.w);
    xa[i][4] = pack_bf2(p1.x, p1.y); xa[i][5] = pack_bf2(p3.x, p3.y);
    xa[i][6] = pack_bf2(p1.z, p1.w); xa[i][7] = pack_bf2(p3.z, p3.w);
  }
  s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
  s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
  s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
  s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
  if ((lane & 3) == 0) {
    s.ssp()[warp * 16 + b0] = s0;
    s.ssp()[warp * 16 + b1] = s1;
  }
  mbar_arrive(s.mbSS());
  return unit_loop<kMaxCA>(a, s, xa, nch, u0, u1, 16 * D, ct);
}

// Phase C, MMA warps: A fragments of g for the quarter of E each unit covers (u / (D/8)), loaded per
// run of units sharing a quarter.
__device__ __forceinline__ Ctr mma_units_c(const DsArgs& a, uint8_t* base, int l, int u0, int u1, Ctr ct) {
  const Smem s{base, &a};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = a.E / 128, qdiv = a.D / 8;
  for (int us = u0; us < u1;) {
    const int q = us / qdiv;
    const int ue = min(u1, (q + 1) * qdiv);
    uint32_t xa[kMaxCC][8];
#pragma unroll
    for (int i = 0; i < kMaxCC; ++i) {
      const int j = min(warp + kMW * i, nch - 1);
      const int k = q * (a.E / 4) + 32 * j + 8 * (lane & 3);   // 8 consecutive channels (permuted fragments)
      const uint4 v0 = __ldcg(reinterpret_cast<const uint4*>(a.g + (size_t)(lane >> 2) * a.E + k));
      const uint4 v1 = __ldcg(reinterpret_cast<const uint4*>(a.g + (size_t)((lane >> 2) + 8) * a.E + k));
      xa[i][0] = v0.x; xa[i][1] = v1.x; xa[i][2] = v0.y; xa[i][3] = v1.y;
      xa[i][4] = v0.z; xa[i][5] = v1.z; xa[i][6] = v0.w; xa[i][7] = v1.w;
    }
    ct = unit_loop<kMaxCC>(a, s, xa, nch, us, ue, 4 * a.E, ct);
    us = ue;
  }
  return ct;
}

// Epilogue thread e = (b = e / 8, n = e % 8): the unit's output element (token b, row n), summed over
// the kMW partials in fixed warp order.
SSM_DEV float reduce_unit(const Smem& s, int useq, int b, int n) {
  const float* sp = s.sred() + (useq % kRB) * (kMW * 128) + ((b >> 3) * 2 + (n & 1)) * 32 + (b & 7) * 4 + (n >> 1);
  float v = 0.f;
#pragma unroll
  for (int w = 0; w < kMW; ++w) v += sp[w * 128];
  return v;
}

// Phase A epilogue warps: z rows -> z; x rows -> conv step + SiLU -> u, window shift, x_proj partial.
__device__ __forceinline__ Ctr epi_units_a(const DsArgs& a, uint8_t* base, int l, int u0, int u1, Ctr ct) {
  const Smem s{base, &a};
  const int e = threadIdx.x - kMW * 32, ew = e >> 5, lane = threadIdx.x & 31;
  const int b = e >> 3, n = e & 7;
  const int B = a.B, E = a.E, P = a.P, K = a.K;
  const int gx0 = (u0 + 1) >> 1;
  // the layer's pointers in registers (stores below may alias the layer table as far as the compiler knows)
  __nv_bfloat16* const cst = a.layers[l].cst;
  __nv_bfloat16* const uo = a.u;
  __nv_bfloat16* const zo = a.z;
  // RMSNorm statistic of the pre-norm (reading Q16, weight 1): 1 / sqrt(mean_d r[b][d]^2 + eps)
  mbar_wait(s.mbSS(), l & 1);
  float ss = 0.f;
#pragma unroll
  for (int w = 0; w < kMW; ++w) ss += s.ssp()[w * 16 + b];
  const float rs = rsqrtf(ss / (float)a.D + a.eps);
  mbar_wait(s.mbX(), l & 1);
  cp_async_wait<0>();
  named_bar_sync(2, kEW * 32);
  float xp[kMaxPT][4];
#pragma unroll
  for (int k = 0; k < kMaxPT; ++k) xp[k][0] = xp[k][1] = xp[k][2] = xp[k][3] = 0.f;
  const int npt = P / 8;
  int ux = 0;
  for (int u = u0; u < u1; ++u, ++ct.seq, ++ct.useq) {
    const bool is_x = (u & 1) == 0;
    const int i = u >> 1, f = 8 * i + n, xi = i - gx0;
    if (e == 0 && u - u0 < 8) stamp(a, l, 16 + (u - u0));
    mbar_wait(&s.ready()[ct.useq % kRB], (ct.useq / kRB) & 1);
    if (e == 0 && u - u0 < 8) stamp(a, l, 24 + (u - u0));
    float v = reduce_unit(s, ct.useq, b, n);
    mbar_arrive(&s.freeb()[ct.useq % kRB]);
    v *= rs;
    if (!is_x) {
      if (b < B) zo[(size_t)b * E + f] = __float2bfloat16_rn(v);
      continue;
    }
    // causal conv step (tap K-1 = this token) + SiLU; the window shifts by one
    const float* cw = s.sxcw() + (xi * 8 + n) * K;
    const uint16_t* wn = s.sxwin() + (xi * 16 + b) * 24 + n;
    const float x = __bfloat162float(__float2bfloat16_rn(v));
    float acc = s.sxcb()[xi * 8 + n];
    for (int j = 0; j < K - 1; ++j) acc = fmaf(cw[j], __uint_as_float((uint32_t)wn[j * 8] << 16), acc);
    acc = fmaf(cw[K - 1], x, acc);
    const __nv_bfloat16 ub = __float2bfloat16_rn(silu<true>(acc));
    __nv_bfloat16* ut = s.utile() + (ux & 1) * 128;
    ut[b * 8 + n] = b < B ? ub : __float2bfloat16_rn(0.f);
    if (b < B) {
      uo[(size_t)b * E + f] = ub;
      uint16_t* cs = reinterpret_cast<uint16_t*>(cst);
      for (int j = 0; j < K - 2; ++j) cs[((size_t)b * (K - 1) + j) * E + f] = wn[(j + 1) * 8];
      cst[((size_t)b * (K - 1) + (K - 2)) * E + f] = __float2bfloat16_rn(x);
    }
    named_bar_sync(2, kEW * 32);
    // x_proj partial of these 8 channels: xp[b][p] += sum_n u[b][n] W_x[p][8i + n]  (m16n8k8)
    const uint32_t a0 = *reinterpret_cast<const uint32_t*>(ut + (lane >> 2) * 8 + 2 * (lane & 3));
    const uint32_t a1 = *reinterpret_cast<const uint32_t*>(ut + ((lane >> 2) + 8) * 8 + 2 * (lane & 3));
    const uint32_t* wx = s.sxw() + xi * npt * 32 + lane;
#pragma unroll
    for (int k = 0; k < kMaxPT; ++k)
      if (ew + kEW * k < npt) mma_1688_bf16(xp[k], a0, a1, wx[(ew + kEW * k) * 32]);
    ++ux;
  }
  // this CTA's x_proj partials -> xacc (fp32 reductions)
  float* xacc = a.xacc + (l & 1) * 16 * P;
#pragma unroll
  for (int k = 0; k < kMaxPT; ++k) {
    const int t = ew + kEW * k;
    if (t < npt) {  // (warp-uniform)
      // lane pairs (tig even, tig + 1) hold 4 consecutive columns of rows br and br + 8: the even lane
      // reduces row br's four, the odd lane row br + 8's four (one 16-B reduction each)
      const bool odd = lane & 1;
      const float o0 = __shfl_xor_sync(0xffffffffu, odd ? xp[k][0] : xp[k][2], 1);
      const float o1 = __shfl_xor_sync(0xffffffffu, odd ? xp[k][1] : xp[k][3], 1);
      const int br = (lane >> 2) + (odd ? 8 : 0), p = 8 * t + 2 * (lane & 2);
      if (br < B) {
        float* dst = xacc + br * P + p;
        if (odd) asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(o0), "f"(o1), "f"(xp[k][2]), "f"(xp[k][3]) : "memory");
        else asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(xp[k][0]), "f"(xp[k][1]), "f"(o0), "f"(o1) : "memory");
      }
    }
  }
  return ct;
}

// Phase C epilogue warps: r += the unit's partial (fp32 reductions; the four K quarters of a row group
// come from different CTAs and are complete at the grid barrier that ends the phase).
__device__ __forceinline__ Ctr epi_units_c(const DsArgs& a, uint8_t* base, int u0, int u1, Ctr ct) {
  const Smem s{base, &a};
  const int e = threadIdx.x - kMW * 32;
  const int b = e >> 3, n = e & 7;
  const int D = a.D;
  float* const r = a.r;
  for (int u = u0; u < u1; ++u, ++ct.seq, ++ct.useq) {
    const int g8 = u % (D / 8);
    mbar_wait(&s.ready()[ct.useq % kRB], (ct.useq / kRB) & 1);
    const float v = reduce_unit(s, ct.useq, b, n);
    mbar_arrive(&s.freeb()[ct.useq % kRB]);
    if (b < a.B) red_add_f32(r + (size_t)b * D + 8 * g8 + n, v);
  }
  return ct;
}

// Phase B (all work threads): dt_proj + softplus + scan step + D skip + gate for this CTA's channels.
__device__ __forceinline__ void phase_b(const DsArgs& a, uint8_t* base, int l, int gb0, int gb1) {
  const Smem s{base, &a};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = a.B, E = a.E, P = a.P, R = a.R;
  const int nch = 8 * (gb1 - gb0), d0 = 8 * gb0, ng = gb1 - gb0;
  const int PS = P + 8;  // smem row stride of the dbc rows: 8 banks shift per token (dt_proj A fragments)
  float* const hglob = a.layers[l].h;
  __nv_bfloat16* const gout = a.g;
  const float* xacc = a.xacc + (l & 1) * 16 * P;
  // u and z rows of this CTA's channels -> shared memory (16-B cp.async pieces of the 2 nch-byte rows)
  const int nit = B * nch;
  for (int i = tid; i < 2 * B * (nch / 8); i += kWork) {
    const int which = i / (B * (nch / 8)), r = i % (B * (nch / 8)), bb = r / (nch / 8), c8 = r % (nch / 8);
    const __nv_bfloat16* src = (which ? a.z : a.u) + (size_t)bb * E + d0 + 8 * c8;
    cp_async16((which ? s.sz() : s.su()) + bb * a.nch_max + 8 * c8, src, true);
  }
  // the summed x_proj rows (dt_low | B | C) -> shared memory by cp.async, all copies in flight at once
  // (rows >= B zero-filled)
  for (int i = tid; i < 16 * (P / 4); i += kWork) {
    const int bb = i / (P / 4), q = i % (P / 4);
    cp_async16(s.sdbc() + bb * PS + 4 * q, xacc + (bb < B ? bb : 0) * P + 4 * q, bb < B);
  }
  cp_async_commit();
  cp_async_wait<0>();
  if (tid == 0) stamp(a, l, 11);
  mbar_wait(s.mbB(), l & 1);
  if (tid == 0) stamp(a, l, 12);
  for (int i = tid; i < nch * 16; i += kWork)
    s.sA()[i] = -ex2_approx(s.salog()[i] * 1.4426950408889634f) * 1.4426950408889634f;  // A log2(e)
  named_bar_sync(1, kWork);
  if (a.bcdt_rmsnorm) {  // weightless RMSNorm of dt_low, B, C per token (Falcon-Mamba, reading Q18)
    for (int bb = warp; bb < B; bb += kMW + kEW) {
      float s0 = 0.f, s1 = 0.f, s2 = 0.f;
      for (int p = lane; p < P; p += 32) {
        const float v = s.sdbc()[bb * PS + p];
        if (p < R) s0 = fmaf(v, v, s0);
        else if (p < R + 16) s1 = fmaf(v, v, s1);
        else s2 = fmaf(v, v, s2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      const float r0 = rsqrtf(s0 / (float)R + a.rms_eps), r1 = rsqrtf(s1 * (1.f / 16.f) + a.rms_eps),
                  r2 = rsqrtf(s2 * (1.f / 16.f) + a.rms_eps);
      __syncwarp();
      for (int p = lane; p < P; p += 32) s.sdbc()[bb * PS + p] *= (p < R ? r0 : p < R + 16 ? r1 : r2);
    }
    named_bar_sync(1, kWork);
  }
  // dt_proj on the tensor pipe: dt[b][ch] = sum_r dt_low[b][r] W_dt[ch][r] (m16n8k16, warp = 8 channels)
  if (warp < ng) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};  // even / odd k16 steps
    const int br = lane >> 2, kq = 2 * (lane & 3);
    const uint2* wb = reinterpret_cast<const uint2*>(s.swdt()) + warp * (R / 16) * 32 + lane;
#pragma unroll 2
    for (int st = 0; st < R / 16; ++st) {
      const float* r0 = s.sdbc() + br * PS + 16 * st + kq;
      const float* r1 = r0 + 8 * PS;
      const uint32_t af[4] = {pack_bf2(r0[0], r0[1]), pack_bf2(r1[0], r1[1]), pack_bf2(r0[8], r0[9]),
                              pack_bf2(r1[8], r1[9])};
      const uint2 w2 = wb[st * 32];
      if (st & 1) mma_16816_bf16(acc2, af, w2.x, w2.y);
      else mma_16816_bf16(acc, af, w2.x, w2.y);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += acc2[q];
    const int ch = 8 * warp + kq;
    float* sdt = s.sdt();
    // softplus with the linear branch above 20; 2-MUFU form (bf16 mode)
    auto sp = [](float x) { return x > 20.f ? x : 0.6931471805599453f * __log2f(1.f + ex2_approx(x * 1.4426950408889634f)); };
    sdt[br * a.nch_max + ch] = sp(acc[0] + s.sbdt()[ch]);
    sdt[br * a.nch_max + ch + 1] = sp(acc[1] + s.sbdt()[ch + 1]);
    sdt[(br + 8) * a.nch_max + ch] = sp(acc[2] + s.sbdt()[ch]);
    sdt[(br + 8) * a.nch_max + ch + 1] = sp(acc[3] + s.sbdt()[ch + 1]);
  }
  named_bar_sync(1, kWork);
  if (tid == 0) stamp(a, l, 13);
  // items (b, ch) with 4 lanes per item, each lane owning 4 of the 16 states (one float4): the h / A rows
  // of the 8 items of a warp are then contiguous 512-B runs in shared and global memory
  // item it = bb nch + ch advances by kWork / 4 per round: (bb, ch) updated without divisions
  const int step_b = (kWork / 4) / nch, step_c = (kWork / 4) % nch;
  int ib = (tid >> 2) / nch, ic = (tid >> 2) % nch;
  for (int task0 = 0; task0 < 4 * nit; task0 += kWork) {
    const int it = (task0 + tid) >> 2, nq = 4 * (tid & 3);
    const bool ok = it < nit;   // (all 4 lanes of an item agree; the shuffles below run warp-wide)
    const int bb = ok ? ib : 0, ch = ok ? ic : 0;
    ib += step_b;
    ic += step_c;
    if (ic >= nch) { ic -= nch; ++ib; }
    const float dt = s.sdt()[bb * a.nch_max + ch];
    const float uq = __bfloat162float(s.su()[bb * a.nch_max + ch]);
    const float du = dt * uq;
    const float4 h4 = *reinterpret_cast<const float4*>(s.sh() + ((size_t)bb * a.nch_max + ch) * 16 + nq);
    const float4 a4 = *reinterpret_cast<const float4*>(s.sA() + ch * 16 + nq);
    const float4 b4 = *reinterpret_cast<const float4*>(s.sdbc() + bb * PS + R + nq);
    const float4 c4 = *reinterpret_cast<const float4*>(s.sdbc() + bb * PS + R + 16 + nq);
    float4 o;  // h_t = exp(dt A) h_{t-1} + dt B_t u_t  (ZOH for A, Euler for B: reading Q1)
    o.x = fmaf(ex2_approx(dt * a4.x), h4.x, du * b4.x);
    o.y = fmaf(ex2_approx(dt * a4.y), h4.y, du * b4.y);
    o.z = fmaf(ex2_approx(dt * a4.z), h4.z, du * b4.z);
    o.w = fmaf(ex2_approx(dt * a4.w), h4.w, du * b4.w);
    float y = c4.x * o.x;
    y = fmaf(c4.y, o.y, y); y = fmaf(c4.z, o.z, y); y = fmaf(c4.w, o.w, y);
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    y += __shfl_xor_sync(0xffffffffu, y, 2);
    if (ok) {
      *reinterpret_cast<float4*>(hglob + ((size_t)bb * E + d0 + ch) * 16 + nq) = o;
      if (nq == 0) {
        y = fmaf(s.sdsk()[ch], uq, y);
        gout[(size_t)bb * E + d0 + ch] = __float2bfloat16_rn(y * silu<true>(__bfloat162float(s.sz()[bb * a.nch_max + ch])));
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) decode_stack_kernel(const __grid_constant__ DsArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Smem s{base, &a};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x, nc = gridDim.x;
  const int D = a.D, E = a.E;
  const int UA = E / 4;                    // in_proj units (2E rows / 8)
  const int UC = D / 2;                    // out_proj units (4 quarters x D/8)
  const int ua0 = part(UA, c, nc), ua1 = part(UA, c + 1, nc);
  const int uc0 = part(UC, c, nc), uc1 = part(UC, c + 1, nc);
  const int gb0 = part(E / 8, c, nc), gb1 = part(E / 8, c + 1, nc);
  const int gx0 = (ua0 + 1) >> 1, gx1 = (ua1 + 1) >> 1;   // x groups of this CTA's in_proj units

  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&s.full()[i], 1);
      mbar_init(&s.empty()[i], kMW * 32);
    }
    for (int i = 0; i < kRB; ++i) {
      mbar_init(&s.ready()[i], kMW * 32);
      mbar_init(&s.freeb()[i], kEW * 32);
    }
    mbar_init(s.mbB(), 1);
    mbar_init(s.mbX(), 1);
    mbar_init(s.mbSS(), kMW * 32);
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------- ring producer (warp kMW + kEW, lane 0): every layer's A units then C units of this
  // CTA in order (cp.async.bulk, L2 evict-first), as far as ring space allows -- weights never
  // depend on activations, so the stream runs ahead across phases, barriers and layers
  if (warp == kMW + kEW) {
    if (lane == 0) {
      Pump* pump = s.pump();
      Pump p{};
      p.nA = ua1 - ua0; p.nC = uc1 - uc0; p.ua0 = ua0; p.uc0 = uc0; p.szA = 16 * D; p.szC = 4 * E;
      p.total = a.L * (p.nA + p.nC);
      *pump = p;
      pump_run(a, s, pump);
    }
    return;
  }

  // ---------------- work threads: MMA warps 0..kMW-1, epilogue warps kMW..kMW+kEW-1
  const bool mw = warp < kMW;
  unsigned nbar = 0;
  Ctr ct{0, 0, 0};
  if (tid == 0) {
    issue_phase_b_prefetch(a, s, a.layers[0], gb0, gb1);
    issue_phase_a_prefetch(a, s, a.layers[0], gx0, gx1);
  }
  if (!mw) issue_window_prefetch(a, s, a.layers[0], gx0, gx1, tid - kMW * 32);

  for (int l = 0; l < a.L; ++l) {
    // ---- A: pre-norm statistic + in_proj + conv step + x_proj partial
    if (tid == 0) stamp(a, l, 0);
    if (mw) ct = mma_units_a(a, base, l, ua0, ua1, ct);
    else ct = epi_units_a(a, base, l, ua0, ua1, ct);
    if (tid == 0) stamp(a, l, 1);
    if (tid == kMW * 32) stamp(a, l, 2);
    grid_sync(a.bar, (++nbar) * nc);
    if (tid == 0) stamp(a, l, 3);
    // ---- B: dt_proj + softplus + scan step + D skip + gate
    phase_b(a, base, l, gb0, gb1);
    if (tid == 0) stamp(a, l, 4);
    grid_sync(a.bar, (++nbar) * nc);
    if (tid == 0) stamp(a, l, 5);
    // ---- C: out_proj (K quarters) -> residual; the next layer's phase-A/B operands prefetched now
    if (l + 1 < a.L) {
      if (tid == 0) {
        issue_phase_b_prefetch(a, s, a.layers[l + 1], gb0, gb1);
        issue_phase_a_prefetch(a, s, a.layers[l + 1], gx0, gx1);
      }
      if (!mw) issue_window_prefetch(a, s, a.layers[l + 1], gx0, gx1, tid - kMW * 32);
    }
    if (c == 0) {
      float* xacc = a.xacc + (l & 1) * 16 * a.P;
      for (int i = tid; i < 16 * a.P; i += kWork) xacc[i] = 0.f;  // re-armed for layer l + 2
    }
    if (mw) ct = mma_units_c(a, base, l, uc0, uc1, ct);
    else ct = epi_units_c(a, base, uc0, uc1, ct);
    if (tid == 0) stamp(a, l, 6);
    if (tid == kMW * 32) stamp(a, l, 7);
    if (l + 1 < a.L) grid_sync(a.bar, (++nbar) * nc);
    if (tid == 0) stamp(a, l, 8);
  }

  // exit: the last CTA out resets the barrier counter for the next launch
  named_bar_sync(1, kWork);
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.bar + 1, 1u) == (unsigned)nc - 1) {
      atomicExch(a.bar, 0u);
      atomicExch(a.bar + 1, 0u);
    }
  }
}

// ---------------------------------------------------------------- weight packing (once per plan)
// B fragments of an 8-row block over a 32-wide k chunk, k permuted inside the chunk: lane L holds
// W[row0 + L/4][k0 + 8 (L%4) + 0..7] and uses elements 0-1 / 2-3 as b0 / b1 of the first k16 step and
// 4-5 / 6-7 as b0 / b1 of the second.  The A fragments use the same permutation (a lane's 8 elements
// of a row are the activations at k0 + 8 (L%4) + 0..7), so both operands load as contiguous 16-B runs
// of row-major data; the dot product over the chunk is unchanged (a permutation of its terms).
__device__ __forceinline__ uint4 bfrag8x32(const __nv_bfloat16* W, int64_t ld, int row, int k0, int lane) {
  return *reinterpret_cast<const uint4*>(W + (int64_t)row * ld + k0 + 8 * (lane & 3));
}

// in_proj [2E][D] -> units (x group i = 2i, z group i = 2i+1) of D/32 chunks
__global__ void pack_wa_kernel(const __nv_bfloat16* __restrict__ w, int E, int D, uint4* __restrict__ out) {
  const int64_t n = (int64_t)(E / 4) * (D / 32) * 32;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(v & 31);
    const int64_t cu = v >> 5;
    const int j = (int)(cu % (D / 32));
    const int u = (int)(cu / (D / 32));
    const int row = ((u & 1) ? E : 0) + 8 * (u >> 1) + (lane >> 2);
    out[v] = bfrag8x32(w, D, row, 32 * j, lane);
  }
}
// out_proj [D][E] -> units (quarter qq, row group g) = qq * D/8 + g of E/128 chunks
__global__ void pack_wc_kernel(const __nv_bfloat16* __restrict__ w, int D, int E, uint4* __restrict__ out) {
  const int64_t n = (int64_t)(D / 2) * (E / 128) * 32;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(v & 31);
    const int64_t cu = v >> 5;
    const int j = (int)(cu % (E / 128));
    const int u = (int)(cu / (E / 128));
    const int qq = u / (D / 8), g = u % (D / 8);
    out[v] = bfrag8x32(w, E, 8 * g + (lane >> 2), qq * (E / 4) + 32 * j, lane);
  }
}
// x_proj [P][E] -> [E/8][P/8][32] u32: {W_x[8t + L/4][8i + 2q], +1}
__global__ void pack_wx_kernel(const __nv_bfloat16* __restrict__ w, int P, int E, uint32_t* __restrict__ out) {
  const int64_t n = (int64_t)(E / 8) * (P / 8) * 32;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(v & 31);
    const int t = (int)((v >> 5) % (P / 8));
    const int i = (int)((v >> 5) / (P / 8));
    out[v] = *reinterpret_cast<const uint32_t*>(w + (int64_t)(8 * t + (lane >> 2)) * E + 8 * i + 2 * (lane & 3));
  }
}
// dt_proj [E][R] -> [E/8][R/16][32] x 8 B: {W_dt[8g + L/4][16s + 2q], +1, [+8], [+9]}
__global__ void pack_wdt_kernel(const __nv_bfloat16* __restrict__ w, int E, int R, uint2* __restrict__ out) {
  const int64_t n = (int64_t)(E / 8) * (R / 16) * 32;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(v & 31);
    const int st = (int)((v >> 5) % (R / 16));
    const int g = (int)((v >> 5) / (R / 16));
    const __nv_bfloat16* p = w + (int64_t)(8 * g + (lane >> 2)) * R + 16 * st + 2 * (lane & 3);
    out[v] = make_uint2(*reinterpret_cast<const uint32_t*>(p), *reinterpret_cast<const uint32_t*>(p + 8));
  }
}

}  // namespace

// ---------------------------------------------------------------- host side
size_t ds_packed_layer_bytes(int D, int E, int R, int P) {
  auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  return al((size_t)2 * E * D * 2) + al((size_t)D * E * 2) + al((size_t)E * P * 2) + al((size_t)E * R * 2);
}

DsGeom ds_geometry(int B, int D, int E, int R, int P, int K, int num_sms) {  // num_sms: grid size
  DsGeom g{};
  g.ok = B >= 1 && B <= 16 && D % 128 == 0 && D / 32 <= kMW * kMaxCA && E % 128 == 0 && E / 128 <= kMW * kMaxCC &&
         R % 16 == 0 && P == R + 32 && P % 8 == 0 && P / 8 <= kEW * kMaxPT && K >= 2 && K <= 4 && num_sms >= 1;
  const int gmax = (E / 8 + num_sms - 1) / num_sms;
  g.nch_max = 8 * gmax;
  auto al = [](int x) { return (x + 127) & ~127; };
  const int sb = al(B * g.nch_max * 64) + al(gmax * (R / 16) * 256) + al(g.nch_max * 64) + al(g.nch_max * 4) * 2;
  const int red = kRB * kMW * 128 * 4;
  const int pbB = al(16 * (P + 8) * 4) + al(16 * g.nch_max * 4) + al(g.nch_max * 16 * 4) + 2 * 16 * g.nch_max * 2;
  const int pbA = kMaxXU * P * 16 + kMaxXU * 8 * 4 * 4 + kMaxXU * 8 * 4 + kMaxXU * 16 * 3 * 8 * 2;
  const int pbz = al(pbB > pbA ? pbB : pbA);
  const int ut = 2 * 16 * 8 * 2;
  const int misc = 1024 + 128;  // mbarriers, pre-norm partials | pump state
  const int fixed = sb + red + pbz + ut + misc;
  const int budget = 227 * 1024 - 1024;  // dynamic smem minus the 1 KB alignment slack
  int ring = (budget - fixed) / 4096 * 4096;
  const int maxunit = 16 * D > 4 * E ? 16 * D : 4 * E;
  if (ring < 2 * maxunit) g.ok = false;
  if ((D / 2 + num_sms - 1) / num_sms > 32 || gmax > kMW + kEW ||
      (E / 4 + num_sms - 1) / num_sms > 2 * kMaxXU - 1)
    g.ok = false;
  g.ring_bytes = ring;
  g.off_sb = ring;
  g.off_red = g.off_sb + sb;
  g.off_pb = g.off_red + red;
  g.off_ut = g.off_pb + pbz;
  g.off_misc = g.off_ut + ut;
  g.smem = g.off_misc + misc + 1024;
  g.scratch_bytes = 3 * (size_t)16 * E * 2 + (size_t)2 * 16 * P * 4 + 64;
  return g;
}

cudaError_t ds_pack_layer(const __nv_bfloat16* w_in, const __nv_bfloat16* w_out, const __nv_bfloat16* w_x,
                          const __nv_bfloat16* w_dt, int D, int E, int R, int P, uint8_t* dst, cudaStream_t s) {
  auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  uint8_t* wa = dst;
  uint8_t* wc = wa + al((size_t)2 * E * D * 2);
  uint8_t* wx = wc + al((size_t)D * E * 2);
  uint8_t* wd = wx + al((size_t)E * P * 2);
  pack_wa_kernel<<<1184, 256, 0, s>>>(w_in, E, D, reinterpret_cast<uint4*>(wa));
  pack_wc_kernel<<<1184, 256, 0, s>>>(w_out, D, E, reinterpret_cast<uint4*>(wc));
  pack_wx_kernel<<<296, 256, 0, s>>>(w_x, P, E, reinterpret_cast<uint32_t*>(wx));
  pack_wdt_kernel<<<296, 256, 0, s>>>(w_dt, E, R, reinterpret_cast<uint2*>(wd));
  return cudaGetLastError();
}

cudaError_t ds_fill_layer(DsLayer* host_entry, const uint8_t* packed, int D, int E, int R, int P,
                          const float* conv_w, const float* conv_b, const float* b_dt, const float* a_log,
                          const float* d_skip, void* cst, float* h) {
  auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  DsLayer& ly = *host_entry;
  ly.wa = packed;
  ly.wc = packed + al((size_t)2 * E * D * 2);
  ly.wxf = reinterpret_cast<const uint32_t*>(ly.wc + al((size_t)D * E * 2));
  ly.wdt = reinterpret_cast<const uint8_t*>(ly.wxf) + al((size_t)E * P * 2);
  ly.conv_w = conv_w;
  ly.conv_b = conv_b;
  ly.b_dt = b_dt;
  ly.a_log = a_log;
  ly.d_skip = d_skip;
  ly.cst = reinterpret_cast<__nv_bfloat16*>(cst);
  ly.h = h;
  return cudaSuccess;
}

size_t ds_layer_entry_bytes() { return sizeof(DsLayer); }

cudaError_t ds_launch(const DsLayer* layers_dev, int L, int B, int D, int E, int R, int P, int K, float eps,
                      int bcdt_rmsnorm, float rms_eps, float* r, uint8_t* scratch, const DsGeom& g, int num_sms,
                      cudaStream_t s, unsigned long long* trace) {
  DsArgs a{};
  a.layers = layers_dev;
  a.L = L; a.B = B; a.D = D; a.E = E; a.R = R; a.P = P; a.K = K;
  a.eps = eps;
  a.bcdt_rmsnorm = bcdt_rmsnorm;
  a.rms_eps = rms_eps;
  a.r = r;
  uint8_t* p = scratch;
  a.g = reinterpret_cast<__nv_bfloat16*>(p); p += (size_t)16 * E * 2;
  a.u = reinterpret_cast<__nv_bfloat16*>(p); p += (size_t)16 * E * 2;
  a.z = reinterpret_cast<__nv_bfloat16*>(p); p += (size_t)16 * E * 2;
  a.xacc = reinterpret_cast<float*>(p); p += (size_t)2 * 16 * P * 4;
  a.bar = reinterpret_cast<unsigned*>(p);
  a.ring_bytes = g.ring_bytes;
  a.nch_max = g.nch_max;
  a.off_sb = g.off_sb;
  a.off_red = g.off_red;
  a.off_pb = g.off_pb;
  a.off_ut = g.off_ut;
  a.off_misc = g.off_misc;
  a.trace = trace;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_stack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_stack_kernel, a);
}

cudaError_t preload_decode_stack() {
  cudaError_t e = cudaFuncSetAttribute(decode_stack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, decode_stack_kernel);
}

int ds_max_active(int smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_stack_kernel, kThreads, smem) != cudaSuccess) return 0;
  return n;
}

}  // namespace ssm
