// decode_mk.cu — persistent whole-stack decode: ONE launch runs one decode token (L = 1) for every
// sequence of the batch through all n_layers pre-norm mixer blocks of a TP=1 stack
// (SURVEY.md §8 rows a1-a11 with M = batch; PAPER.md:151-174 the mixer, 276-287 the cache carried
// into decode, 545 "TPOT ... memory footprint and bandwidth").
//
// Why one kernel: a decode token streams every layer's weights once (Mamba-2.8B: 82.6 MB/layer,
// 5.3 GB/token at bf16) and little else, so the step is HBM-bound -- but as a chain of small
// kernels each launch pays a ramp-up/drain of the HBM stream (~2.5 us per launch,
// profiles/r01_stream_probe_21.txt) and the latency-bound middle of a layer (conv, x_proj,
// decode step) leaves HBM idle.  Here, on a persistent grid of one CTA per SM:
//   * warp 8 streams the CTA's share of every layer's packed W_in / W_out tiles (16 KB, 1D bulk
//     copies) into a shared-memory ring, with L2 prefetches running about one phase ahead, and
//     never waits for activations: weights do not depend on them;
//   * warp 9 bulk-loads the B operands (k-blocks of the bf16 residual / of the gated scan
//     output g) into a second ring as soon as their producers have published them;
//   * warps 0-7 run the phases of each layer.
// Cross-CTA dependencies are per-tile readiness counters (monotonic, in the workspace), not grid
// barriers: a phase waits only for the tiles it reads.  Per layer (epoch e):
//   A  in_proj (a1): stream-K over W_in tiles; fp32 partials red.add into xzT [2Ek][BP]; after a
//      row tile's partials: cnt_in[rt] += 1.
//   B  (waits cnt_in of its x / z row tiles) conv step + SiLU (a2) for the CTA's channels, the
//      cache window shifted in place; x_proj partial (a3, mma.sync) red.add into dbcT; cnt_x += 1.
//      The pre-norm RMSNorm (weight 1, reading Q16) is applied here: 1/rms(row) factors out of
//      the in_proj contraction, so x and z are scaled after the GEMM.
//   C  (waits cnt_x: the one all-to-all of the layer) decode step (a4-a7): dt_low/B/C (+ Falcon
//      RMSNorm), dt_proj (mma.sync) + softplus, one ZOH/Euler scan step with h in place, D skip,
//      SiLU(z) gate -> gT; rdy_g[k-block] += 1.
//   D  out_proj (a8): stream-K over W_out tiles (B = gT k-blocks, loaded by warp 9 once ready);
//      partials red.add into residT [D][BP] (TP=1: the residual add of a9, reading Q13).  The
//      last contributor of a residual row tile finalises it: bf16 copy (next in_proj's B),
//      sums of squares (next pre-norm), output rows after the last layer; rdy_res[rt] = e + 1.
// The decode GEMMs have N = batch <= 32 columns: 16 flop per weight byte, bound by the weight
// stream (HBM), not by the tensor pipe; mma.sync m16n8k16 from shared memory keeps the consumers
// ahead of the stream without TMEM allocation or UMMA descriptors.
#include "common.cuh"
#include "internal.h"

namespace ssm {
namespace {

constexpr int MK_CONSUMERS = 256;              // 8 consumer warps
constexpr int MK_WPROD = MK_CONSUMERS / 32;    // warp 8: weight stream
constexpr int MK_BPROD = MK_WPROD + 1;         // warp 9: B-operand stream
constexpr int MK_MMA = MK_BPROD + 1;           // warp 10: tcgen05.mma issue (one elected lane)
constexpr int MK_THREADS = MK_CONSUMERS + 96;
constexpr int MK_TILE = 16384;                 // one packed 128 x 64 bf16 weight tile
constexpr int MK_N = 16;                       // d_state
constexpr int MK_KH = 3;                       // decode-step items per thread with loads issued early
constexpr uint64_t MK_TIMEOUT_NS = 4000000000ull;  // 4 s: a decode token takes ~1 ms
constexpr float LOG2E = 1.4426950408889634f;
__device__ int g_mk_testwait = 1;  // experiment switch: mbarrier.test_wait (1) or try_wait (0) polling

struct MkLayout {
  uint32_t ring, bars, bring, wx, wdt, sd, sdl, su, sub, sdt, sa2, sbdt, sdsk, scb, scw, sal, sconv, srs, sns, red,
      flag, total;
};

__host__ __device__ inline uint32_t al128(uint32_t x) { return (x + 127u) & ~127u; }
// one B k-block: BP rows (batch) x 64 k bf16, K-major, SWIZZLE_128B image (chunk j of row b at j ^ (b & 7))
__host__ __device__ inline uint32_t mk_bsz(int BP) { return (uint32_t)BP * 128u; }

// Shared-memory map.  Row pitches are 16 B x odd so eight ldmatrix row addresses hit distinct
// 16-B bank groups.  sD / sDl (phase C) alias sWx (phase B operand, dead by then).
__host__ __device__ inline MkLayout mk_layout(int BP, int P, int R, int ncmax, int ring, int nbr) {
  MkLayout L{};
  uint32_t o = 0;
  L.ring = o; o += al128((uint32_t)ring * MK_TILE);
  L.bars = o; o += al128((uint32_t)(2 * ring + 2 * nbr + 8) * 8);
  o = (o + 1023u) & ~1023u;  // UMMA SW128 operands: 1024-B aligned
  L.bring = o; o += al128((uint32_t)nbr * mk_bsz(BP));
  L.wx = o;
  const uint32_t wx_end = o + al128((uint32_t)P * (ncmax + 8) * 2);
  L.sd = o;
  L.sdl = L.sd + al128((uint32_t)P * BP * 4);
  const uint32_t c_end = L.sdl + al128((uint32_t)BP * (R + 8) * 2);
  o = wx_end > c_end ? wx_end : c_end;
  L.wdt = o; o += al128((uint32_t)ncmax * (R + 8) * 2);
  L.su = o; o += al128((uint32_t)BP * ncmax * 4);
  L.sub = o; o += al128((uint32_t)BP * (ncmax + 8) * 2);
  L.sdt = o; o += al128((uint32_t)BP * ncmax * 4);
  L.sa2 = o; o += al128((uint32_t)MK_N * ncmax * 4);
  L.sbdt = o; o += al128((uint32_t)ncmax * 4);
  L.sdsk = o; o += al128((uint32_t)ncmax * 4);
  L.scb = o; o += al128((uint32_t)ncmax * 4);
  L.scw = o; o += al128((uint32_t)ncmax * 4 * 4);
  L.sal = o; o += al128((uint32_t)ncmax * MK_N * 4);
  L.sconv = o; o += al128((uint32_t)BP * 3 * ncmax * 2);
  L.srs = o; o += al128((uint32_t)BP * 4);
  L.sns = o; o += al128((uint32_t)BP * 3 * 4);
  L.red = o; o += al128(256u * 4 + 16);
  L.flag = o; o += 128;
  L.total = o + 1024;  // + alignment slack of the dynamic shared memory base
  return L;
}

SSM_DEV void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
SSM_DEV void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// Element index of (k, b) in a B operand stored as K-major SW128 k-blocks [K/64][BP][64].
template <int BP>
SSM_DEV int64_t mk_bidx(int k, int b) {
  return ((int64_t)(k >> 6) * BP + b) * 64 + ((((k >> 3) & 7) ^ (b & 7)) << 3) + (k & 7);
}
SSM_DEV void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
SSM_DEV void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
SSM_DEV void bulk_load_l2keep(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
SSM_DEV float bf16r(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
SSM_DEV bool mk_err(const unsigned* err) { return *reinterpret_cast<const volatile unsigned*>(err) != 0u; }
SSM_DEV uint32_t ld_acquire_gpu_u32(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SSM_DEV uint32_t ld_relaxed_gpu_u32(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SSM_DEV void st_release_gpu_u32(unsigned* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SSM_DEV uint32_t atom_add_acq_rel_gpu(unsigned* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
SSM_DEV bool reached(uint32_t v, uint32_t target) { return (int32_t)(v - target) >= 0; }

// CTAs owning elements [lo, hi) when T elements are split as [c T / G, (c+1) T / G).
SSM_DEV int mk_owners(int lo, int hi, int T, int G) {
  if (hi <= lo) return 0;
  if (T < G) return hi - lo;  // one element per non-empty CTA
  const int a = (int)(((int64_t)(lo + 1) * G - 1) / T), b = (int)(((int64_t)hi * G - 1) / T);
  return b - a + 1;
}

// Spin until *p >= target (acquire); false (error word raised) on timeout or a raised error.
SSM_DEV bool mk_poll(const unsigned* p, uint32_t target, unsigned* err, uint64_t t0) {
  uint32_t n = 0;
  while (!reached(ld_acquire_gpu_u32(p), target)) {
    __nanosleep(64);  // back off: pollers must not starve the L2 slice of the producers' atomics
    if ((++n & 63u) == 0u) {
      if (mk_err(err)) return false;
      if (globaltimer() - t0 > MK_TIMEOUT_NS) {
        atomicExch(err, 3u);
        return false;
      }
    }
  }
  return true;
}

// mbarrier wait that gives up (and raises the error word) instead of hanging the GPU.
// Non-blocking probe of an mbarrier phase (mbarrier.test_wait never suspends the thread).
SSM_DEV bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

SSM_DEV bool mk_wait(uint64_t* bar, uint32_t parity, unsigned* err, uint64_t t0) {
  uint32_t n = 0;
  while (!((g_mk_testwait) ? mbar_test_wait(bar, parity) : mbar_try_wait(bar, parity))) {
    if (n > 4) __nanosleep(64);  // long waits: leave the issue slots to the working warps
    if ((++n & 255u) == 0u) {
      if (mk_err(err)) return false;
      if (globaltimer() - t0 > MK_TIMEOUT_NS) {
        atomicExch(err, 2u);
        return false;
      }
    }
  }
  return true;
}

// Warp-wide wait: one lane polls the mbarrier (32 pollers per warp would crowd the SM's
// synchronisation unit that also services the producers' arrivals), the warp then converges.
SSM_DEV void mk_wait_warp(uint64_t* bar, uint32_t parity, unsigned* err, uint64_t t0) {
  // every lane probes (converged): a lone polling lane with its warp parked at __syncwarp crawls
  uint32_t n = 0;
  while (!__all_sync(0xffffffffu, mbar_test_wait(bar, parity))) {
    if (n > 4) __nanosleep(32);
    if ((++n & 255u) == 0u) {
      if (mk_err(err)) return;
      if (globaltimer() - t0 > MK_TIMEOUT_NS) {
        if ((threadIdx.x & 31) == 0) atomicExch(err, 2u);
        return;
      }
    }
  }
}

// Grid-wide barrier of the consumer warps (kernel start only).  Monotonic arrival counter: this
// CTA's arrival `old` belongs to round old / grid -- no reset between launches.
SSM_DEV void mk_grid_sync(unsigned long long* bar, unsigned* err, uint64_t t0) {
  named_bar_sync(1, MK_CONSUMERS);
  if (threadIdx.x < 32) {  // warp 0 arrives and polls, converged (lane 0 alone would crawl)
    unsigned long long target = 0;
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned long long G = gridDim.x;
      const unsigned long long old = atomicAdd(bar, 1ull);
      target = (old / G + 1ull) * G;
    }
    target = __shfl_sync(0xffffffffu, target, 0);
    uint32_t n = 0;
    while (true) {
      const bool done = threadIdx.x == 0 ? ld_acquire_gpu_u64(bar) >= target : true;
      if (__all_sync(0xffffffffu, done)) break;
      if ((++n & 63u) == 0u) {
        const bool bad = mk_err(err) || globaltimer() - t0 > MK_TIMEOUT_NS;
        if (__any_sync(0xffffffffu, bad)) {
          if (threadIdx.x == 0) atomicExch(err, 1u);
          break;
        }
      }
    }
    if (threadIdx.x == 0) __threadfence();
    __syncwarp();
  }
  named_bar_sync(1, MK_CONSUMERS);
}

// experiment-only timeline: stamp k of layer l on this CTA
SSM_DEV void mk_stamp(const MkParams& p, int l, int k) {
  if (p.trace) p.trace[((size_t)blockIdx.x * p.n_layers + l) * 32 + k] = globaltimer();
}

// L2 prefetch of a contiguous byte range (64 KB requests)
SSM_DEV void mk_prefetch(const void* base, size_t off, size_t bytes) {
  const char* b = reinterpret_cast<const char*>(base) + off;
  for (size_t o = 0; o < bytes; o += 65536) prefetch_l2(b + o, (uint32_t)(bytes - o < 65536 ? bytes - o : 65536));
}

struct Rings {
  uint64_t *full, *empty, *bfull, *bempty, *start, *afull, *aempty;
  int ring, nbr;
  uint32_t tmem;
};

// Consumer side of one GEMM phase over units [ub, ue) (unit u = row tile u / nkb, k-block
// u % nkb): the MMA warp accumulates each row tile's units in a TMEM accumulator (128 lanes x BP
// fp32 columns, double-buffered); here the 8 consumer warps drain it -- warp w reads TMEM lane
// group w % 4 and column half w / 4 -- and red.add the partials into out [rows][BP], then
// on_flush(rt) runs on all consumer threads.
template <int BP, typename F>
SSM_DEV void mk_epi(const Rings& rg, uint32_t& tc, int ub, int ue, int nkb, float* out, unsigned* err, uint64_t t0,
                    F&& on_flush) {
  constexpr int HB = BP / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int eg = warp & 3, half = warp >> 2;
  if (ue <= ub) return;
  for (int rt = ub / nkb; rt <= (ue - 1) / nkb; ++rt, ++tc) {
    const int buf = tc & 1;
    mk_wait_warp(&rg.afull[buf], (tc >> 1) & 1u, err, t0);
    tc_fence_after();
    const uint32_t ta = rg.tmem + ((uint32_t)(eg * 32) << 16) + (uint32_t)(buf * 32 + half * HB);
    float v[HB];
    if constexpr (HB == 8) {
      uint32_t r[8];
      tmem_ld_32x32b_x8(ta, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
    } else {
      uint32_t r[16];
      tmem_ld_32x32b_x16(ta, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&rg.aempty[buf]);
    float* o = out + (int64_t)(rt * 128 + eg * 32 + lane) * BP + half * HB;
#pragma unroll
    for (int j = 0; j < HB; j += 4) red_add_v4(o + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
    on_flush(rt);
  }
}

// Consumers stage the B operand of a whole GEMM phase (the k-block of every unit [ub, ue), in
// unit order, into the B ring; the ring holds a whole phase) right after the grid barrier that
// completed it: one round trip of 16-B loads for all units, then one arrival per slot for the
// MMA warp.  (Bulk copies issued one by one from a single lane measured ~0.3 us per 2 KB copy
// here; the 256 consumer threads have all loads in flight at once.)
template <int BP>
SSM_DEV void mk_stage_b(unsigned char* smem, const MkLayout& L, const Rings& rg, uint32_t& bitc, int ub, int ue,
                        int nkb, const __nv_bfloat16* src, unsigned* err, uint64_t t0, int dbg = 0,
                        unsigned long long* dbg_tr = nullptr) {
  const int tid = threadIdx.x;
  const int n = ue - ub;
  if (n <= 0) return;
  constexpr int PPT = BP * 128 / 16;  // 16-B pieces per k-block tile
  if (tid < 32 && !(dbg & 256)) {
    // slots free (the MMAs of their previous use completed): warp 0 probes up to 32 slots at once
    // and stays converged (a lone polling lane with its warp parked at a barrier crawled)
    const unsigned long long tw = clock64();
    unsigned long long tries = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + (int)tid;
      const uint32_t b = bitc + j;
      bool ok = j >= n;
      while (!__all_sync(0xffffffffu, ok)) {
        if (!ok) ok = mbar_test_wait(&rg.bempty[b % rg.nbr], ((b / rg.nbr) & 1u) ^ 1u);
        ++tries;
      }
    }
    if (dbg_tr && tid == 0) { dbg_tr[0] = clock64() - tw; dbg_tr[1] = tries; }
  }
  named_bar_sync(1, MK_CONSUMERS);
  const int tot = n * PPT;
  for (int q0 = tid; q0 < tot; q0 += 8 * MK_CONSUMERS) {
    uint4 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int q = q0 + e * MK_CONSUMERS;
      if (q < tot) {
        const int j = q / PPT, r = q % PPT;
        const int kb = (ub + j) % nkb;
        v[e] = __ldcg(reinterpret_cast<const uint4*>(src + (int64_t)kb * BP * 64) + r);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int q = q0 + e * MK_CONSUMERS;
      if (q < tot) {
        const int j = q / PPT, r = q % PPT;
        *reinterpret_cast<uint4*>(smem + L.bring + (size_t)((bitc + j) % rg.nbr) * mk_bsz(BP) + r * 16) = v[e];
      }
    }
  }
  fence_proxy_async();  // generic smem writes -> tcgen05.mma (async proxy) reads
  named_bar_sync(1, MK_CONSUMERS);
  if (tid < 32)
    for (int j = tid; j < n; j += 32) mbar_arrive(&rg.bfull[(bitc + j) % rg.nbr]);
  bitc += n;
}

template <int BP>
__global__ void __launch_bounds__(MK_THREADS, 1) decode_mk_kernel(const MkParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const MkLayout L = mk_layout(BP, p.P, p.R, p.ncmax, p.ring, p.nbr);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int B = p.B, D = p.D, Ek = p.Ek, R = p.R, P = p.P, K = p.K;
  const MkCnt CN = mk_cnt_layout(D, Ek);
  Rings rg;
  rg.full = reinterpret_cast<uint64_t*>(smem + L.bars);
  rg.empty = rg.full + p.ring;
  rg.bfull = rg.empty + p.ring;
  rg.bempty = rg.bfull + p.nbr;
  rg.start = rg.bempty + p.nbr;
  rg.afull = rg.start + 1;
  rg.aempty = rg.afull + 2;
  rg.ring = p.ring;
  rg.nbr = p.nbr;
  const uint64_t t0 = globaltimer();
  if (tid == 0) {
    for (int i = 0; i < p.ring; ++i) {
      mbar_init(&rg.full[i], 1);
      mbar_init(&rg.empty[i], 1);   // freed by tcgen05.commit
    }
    for (int i = 0; i < p.nbr; ++i) {
      mbar_init(&rg.bfull[i], 1);
      mbar_init(&rg.bempty[i], 1);
    }
    mbar_init(rg.start, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&rg.afull[i], 1);
      mbar_init(&rg.aempty[i], MK_CONSUMERS / 32);
    }
    fence_barrier_init();
  }
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.flag + 64);
  if (warp == MK_MMA) tmem_alloc(tmem_slot, 64);  // two BP(<=32)-column fp32 accumulators
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  rg.tmem = *tmem_slot;

  // this CTA's share of each phase (identical for every layer)
  const int n_rt1 = 2 * Ek / 128, nkb1 = D / 64, U1 = n_rt1 * nkb1;
  const int n_rt4 = D / 128, nkb4 = Ek / 64, U4 = n_rt4 * nkb4;
  const int u0 = (int)((int64_t)cta * U1 / G), u1 = (int)((int64_t)(cta + 1) * U1 / G);
  const int v0 = (int)((int64_t)cta * U4 / G), v1 = (int)((int64_t)(cta + 1) * U4 / G);
  const int gr0 = cta * p.ngrp / G, gr1 = (cta + 1) * p.ngrp / G;
  const int c0 = gr0 * 16, nc = (gr1 - gr0) * 16;
  const uint32_t e0 = p.ep[cta];  // layers completed since bind (same on every CTA)
  unsigned* cnt = p.cnt;
  const uint32_t bsz = mk_bsz(BP);

  if (warp == MK_WPROD) {  // ---------------- weight stream (warp-uniform; lane 0 issues)
    if (!(p.dbg & 2)) {
      const bool pf = !(p.dbg & 4);
      // L2 prefetches about one phase ahead of the ring (W_out(l) while the ring fills with
      // W_in(l); W_in(l+1) while it fills with W_out(l)): HBM keeps streaming through the
      // latency-bound phases; the ring then refills from L2.
      const size_t in_lo = (size_t)u0 * MK_TILE, in_bytes = (size_t)(u1 - u0) * MK_TILE;
      const size_t out_lo = (size_t)v0 * MK_TILE, out_bytes = (size_t)(v1 - v0) * MK_TILE;
      const bool ld = lane == 0;
      if (p.n_layers > 0 && pf && ld) mk_prefetch(p.layers[0].w_in_pk, in_lo, in_bytes);
      uint32_t it = 0;
      for (int l = 0; l < p.n_layers; ++l) {
        const MkLayer& Ly = p.layers[l];
        if (ld) mk_stamp(p, l, 12);
        if (pf && ld) mk_prefetch(Ly.w_out_pk, out_lo, out_bytes);
        if (nc > 0)  // the decode step's h rows: into L2 now, read in phase B
          for (int b = lane; b < B; b += 32) prefetch_l2(Ly.h + ((int64_t)b * Ek + c0) * MK_N, (uint32_t)nc * MK_N * 4);
        for (int u = u0; u < u1; ++u, ++it) {
          const int s = it % p.ring;
          mk_wait_warp(&rg.empty[s], ((it / p.ring) & 1u) ^ 1u, p.err, t0);
          if (mk_err(p.err)) return;
          if (ld) {
            mbar_arrive_expect_tx(&rg.full[s], MK_TILE);
            bulk_load_evict_first(smem + L.ring + (size_t)s * MK_TILE,
                                  reinterpret_cast<const char*>(Ly.w_in_pk) + (int64_t)u * MK_TILE, MK_TILE, &rg.full[s]);
          }
          __syncwarp();
        }
        if (ld) mk_stamp(p, l, 13);
        if (l + 1 < p.n_layers && pf && ld) mk_prefetch(p.layers[l + 1].w_in_pk, in_lo, in_bytes);
        for (int v = v0; v < v1; ++v, ++it) {
          const int s = it % p.ring;
          mk_wait_warp(&rg.empty[s], ((it / p.ring) & 1u) ^ 1u, p.err, t0);
          if (mk_err(p.err)) return;
          if (ld) {
            mbar_arrive_expect_tx(&rg.full[s], MK_TILE);
            bulk_load_evict_first(smem + L.ring + (size_t)s * MK_TILE,
                                  reinterpret_cast<const char*>(Ly.w_out_pk) + (int64_t)v * MK_TILE, MK_TILE, &rg.full[s]);
          }
          __syncwarp();
        }
      }
    }
    return;
  }

  if (warp == MK_BPROD) return;  // (spare warp)

  if (warp == MK_MMA) {  // ---------------- tcgen05.mma issue
    // The whole warp runs the (warp-uniform) schedule; one elected lane issues the MMAs and the
    // commits that free the ring slots when the MMAs reading them complete.
    const uint32_t idesc = umma_idesc_bf16(128, BP);
    const uint64_t ring_desc = umma_desc_sw128(smem_u32(smem + L.ring));
    const uint64_t bring_desc = umma_desc_sw128(smem_u32(smem + L.bring));
    uint32_t it = 0, bit = 0, tc = 0;
    auto phase = [&](int ub, int ue, int nkb, int l, int k0) {
      bool first = true;
      int buf = 0;
      unsigned long long wf = 0, wb = 0, w_mma = 0, w_com = 0, w_tot = 0;
      const unsigned long long l0_ = clock64();
      for (int u = ub; u < ue; ++u) {
        const int kk = u % nkb;
        if (u == ub || kk == 0) {
          buf = tc & 1;
          mk_wait_warp(&rg.aempty[buf], ((tc >> 1) & 1u) ^ 1u, p.err, t0);
          tc_fence_after();
          first = true;
        }
        const int s = it % p.ring, bs = bit % p.nbr;
        const unsigned long long c0_ = clock64();
        if (!(p.dbg & 2)) mk_wait_warp(&rg.full[s], (it / p.ring) & 1u, p.err, t0);
        const unsigned long long c1_ = clock64();
        if (u == ub) {  // the consumers stage (and arrive on) every slot of the phase at once
          const uint32_t bl = bit + (uint32_t)(ue - ub - 1);
          mk_wait_warp(&rg.bfull[bl % p.nbr], (bl / p.nbr) & 1u, p.err, t0);
        }
        wf += c1_ - c0_;
        wb += clock64() - c1_;
        if (!(p.dbg & 64)) tc_fence_after();
        if (lane == 0 && u == ub) mk_stamp(p, l, k0);
        if (lane == 0 && u == ue - 1) mk_stamp(p, l, k0 + 1);
        const uint64_t ad = ring_desc + (uint64_t)(((uint32_t)s * MK_TILE) >> 4);
        const uint64_t bd = bring_desc + (uint64_t)(((uint32_t)bs * bsz) >> 4);
        const unsigned long long q0_ = clock64();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            if (!(p.dbg & 16)) umma_bf16(rg.tmem + (uint32_t)(buf * 32), ad + (uint64_t)(ks * 2), bd + (uint64_t)(ks * 2), idesc,
                      (first && ks == 0) ? 0u : 1u);
          const unsigned long long q1_ = clock64();
          if (!(p.dbg & 256)) {
            umma_commit(&rg.empty[s]);
            umma_commit(&rg.bempty[bs]);
          }
          const unsigned long long q2_ = clock64();
          w_mma += q1_ - q0_;
          w_com += q2_ - q1_;
        }
        __syncwarp();
        w_tot += clock64() - q0_;
        first = false;
        ++it;
        ++bit;
        if (u == ue - 1 || kk == nkb - 1) {
          if (elect_one()) umma_commit(&rg.afull[buf]);
          __syncwarp();
          ++tc;
        }
      }
      if (p.trace) {
        w_mma = __shfl_sync(0xffffffffu, w_mma, __ffs(__ballot_sync(0xffffffffu, w_mma != 0)) - 1 < 0 ? 0 : __ffs(__ballot_sync(0xffffffffu, w_mma != 0)) - 1);
      }
      if (lane == 0 && p.trace) {
        p.trace[((size_t)blockIdx.x * p.n_layers + l) * 32 + k0 + 6] = wf;
        p.trace[((size_t)blockIdx.x * p.n_layers + l) * 32 + k0 + 7] = wb;
        if (k0 == 24) {
          p.trace[((size_t)blockIdx.x * p.n_layers + l) * 32 + 10] = w_mma;
          p.trace[((size_t)blockIdx.x * p.n_layers + l) * 32 + 11] = w_tot;
          p.trace[((size_t)blockIdx.x * p.n_layers + l) * 32 + 14] = clock64() - l0_;
        }
      }
    };
    for (int l = 0; l < p.n_layers; ++l) {
      phase(u0, u1, nkb1, l, 24);
      phase(v0, v1, nkb4, l, 20);
    }
    tc_fence_before();
    named_bar_sync(2, MK_CONSUMERS + 32);  // every accumulator drained by the consumers
    tc_fence_after();
    tmem_dealloc(rg.tmem, 64);
    return;
  }

  // ---------------------------------------------------- consumers (warps 0-7)
  const int ncm = p.ncmax;
  const int LDX = ncm + 8, LDR = R + 8;
  __nv_bfloat16* sWx = reinterpret_cast<__nv_bfloat16*>(smem + L.wx);
  __nv_bfloat16* sWdt = reinterpret_cast<__nv_bfloat16*>(smem + L.wdt);
  float* sD = reinterpret_cast<float*>(smem + L.sd);
  __nv_bfloat16* sDl = reinterpret_cast<__nv_bfloat16*>(smem + L.sdl);
  float* su = reinterpret_cast<float*>(smem + L.su);
  __nv_bfloat16* sub = reinterpret_cast<__nv_bfloat16*>(smem + L.sub);
  float* sdt = reinterpret_cast<float*>(smem + L.sdt);
  float* sA2 = reinterpret_cast<float*>(smem + L.sa2);
  float* sBdt = reinterpret_cast<float*>(smem + L.sbdt);
  float* sDsk = reinterpret_cast<float*>(smem + L.sdsk);
  float* sCb = reinterpret_cast<float*>(smem + L.scb);
  float* sCw = reinterpret_cast<float*>(smem + L.scw);                       // [ncm][K]
  float* sAl = reinterpret_cast<float*>(smem + L.sal);                       // [ncm][16] raw a_log
  __nv_bfloat16* sConv = reinterpret_cast<__nv_bfloat16*>(smem + L.sconv);  // [B][K-1][ncm]
  float* sRS = reinterpret_cast<float*>(smem + L.srs);
  float* sNS = reinterpret_cast<float*>(smem + L.sns);
  float* sRed = reinterpret_cast<float*>(smem + L.red);
  volatile int* sFlag = reinterpret_cast<volatile int*>(smem + L.flag);
  const int g = lane >> 2, t = lane & 3, m8 = lane >> 3, r8 = lane & 7;
  const int nI = B * nc;                         // (b, channel) items of this CTA, channel fastest
  const int nx = G < p.ngrp ? G : p.ngrp;        // CTAs with channels (x_proj contributors)
  const bool st0 = tid == 0;

  for (int i = tid; i < BP * LDX; i += MK_CONSUMERS) sub[i] = __float2bfloat16_rn(0.f);  // rows >= B stay 0
  // residual stream in: residT[d][b] = resid[b][d], residB = bf16, per-CTA sums of squares
  {
    const int d0 = (int)((int64_t)cta * D / G), d1 = (int)((int64_t)(cta + 1) * D / G);
    float s = 0.f;
    const int b = tid % BP;
    for (int i = d0 * BP + tid; i < d1 * BP; i += MK_CONSUMERS) {  // thread's column b is fixed
      const int d = i / BP;
      const float v = b < B ? p.resid[(int64_t)b * D + d] : 0.f;
      p.residT[i] = v;
      p.residB[mk_bidx<BP>(d, b)] = __float2bfloat16_rn(v);
      s = fmaf(v, v, s);
    }
    sRed[tid] = s;
    named_bar_sync(1, MK_CONSUMERS);
    if (tid < BP) {
      float a = 0.f;
      for (int j = tid; j < MK_CONSUMERS; j += BP) a += sRed[j];
      p.ssP[(int64_t)cta * BP + tid] = a;
    }
    __threadfence();
    fence_proxy_async_global();
  }
  mk_grid_sync(p.bar, p.err, t0);


  uint32_t tc = 0;    // accumulator tiles drained (same sequence as the MMA warp)
  uint32_t bitc = 0;  // B-ring position (same sequence as the MMA warp)
  for (int l = 0; l < p.n_layers; ++l) {
    const MkLayer Ly = p.layers[l];
    const uint32_t e = e0 + l;
    if (st0) mk_stamp(p, l, 0);
    // ================= phase A: in_proj (a1)
    if (nc > 0) {  // phase B/C operands of this CTA's channels -> smem, one cp.async group
      const int cpr = nc / 8;
      for (int q = tid; q < P * cpr; q += MK_CONSUMERS) {
        const int row = q / cpr, j = q % cpr;
        cp_async16(sWx + row * LDX + j * 8, Ly.w_x + (int64_t)row * Ek + c0 + j * 8, true);
      }
      for (int q = tid; q < B * (K - 1) * cpr; q += MK_CONSUMERS) {  // conv window (owner data)
        const int row = q / cpr, j = q % cpr;
        cp_async16(sConv + row * ncm + j * 8, Ly.conv + (int64_t)row * Ek + c0 + j * 8, true);
      }
      for (int q = tid; q < nc * K / 4; q += MK_CONSUMERS) cp_async16(sCw + q * 4, Ly.conv_w + (int64_t)c0 * K + q * 4, true);
      for (int q = tid; q < nc * MK_N / 4; q += MK_CONSUMERS)
        cp_async16(sAl + q * 4, Ly.a_log + (int64_t)c0 * MK_N + q * 4, true);
      for (int q = tid; q < nc / 4; q += MK_CONSUMERS) {
        cp_async16(sCb + q * 4, Ly.conv_b + c0 + q * 4, true);
        cp_async16(sBdt + q * 4, Ly.b_dt + c0 + q * 4, true);
        cp_async16(sDsk + q * 4, Ly.d_skip + c0 + q * 4, true);
      }
    }
    cp_async_commit();
    if (st0) mk_stamp(p, l, 1);
    mk_stage_b<BP>(smem, L, rg, bitc, u0, u1, nkb1, (p.dbg & 32) ? Ly.w_in_pk : p.residB, p.err, t0, p.dbg,
                   p.trace ? p.trace + ((size_t)cta * p.n_layers + l) * 32 + 28 : nullptr);
    if (st0) mk_stamp(p, l, 23);
    mk_epi<BP>(rg, tc, u0, u1, nkb1, p.xzT, p.err, t0, [&](int) {});
    if (st0) mk_stamp(p, l, 2);
    __threadfence();
    mk_grid_sync(p.bar, p.err, t0);  // xzT complete
    if (st0) mk_stamp(p, l, 3);

    // ================= phase B: conv step + SiLU (a2), x_proj partial (a3)
    if (nc > 0) {  // W_dt rows of this CTA's channels (phase C operand)
      const int cpr = R / 8;
      for (int q = tid; q < nc * cpr; q += MK_CONSUMERS) {
        const int c = q / cpr, j = q % cpr;
        cp_async16(sWdt + c * LDR + j * 8, Ly.w_dt + (int64_t)(c0 + c) * R + j * 8, true);
      }
    }
    cp_async_commit();
    if (cta == 0) {
      // accumulators of epoch e+1: their readers (phases B, C of layer l-1) are behind two grid
      // barriers, their writers (this layer's finalisers; the next layer's x_proj) ahead of one
      for (int i = tid; i < P * BP; i += MK_CONSUMERS) p.dbcT[(size_t)((e + 1) & 1) * P * BP + i] = 0.f;
      if (tid < BP) p.ss[((e + 1) & 1) * BP + tid] = 0.f;
    }
    float zv[MK_KH], hs[MK_KH][MK_N];
    if (nc > 0) {
      // h of this thread's decode-step items (owner data, L2-prefetched) -- before any wait
#pragma unroll
      for (int k = 0; k < MK_KH; ++k) {
        const int i = tid + k * MK_CONSUMERS;
#pragma unroll
        for (int n = 0; n < MK_N; ++n) hs[k][n] = 0.f;
        if (i < nI) {
          const int c = i % nc, b = i / nc, d = c0 + c;
          const float4* hp = reinterpret_cast<const float4*>(Ly.h + ((int64_t)b * Ek + d) * MK_N);
#pragma unroll
          for (int n = 0; n < MK_N; n += 4) {
            const float4 v = __ldcg(hp + n / 4);
            hs[k][n] = v.x; hs[k][n + 1] = v.y; hs[k][n + 2] = v.z; hs[k][n + 3] = v.w;
          }
        }
      }
      float xv[MK_KH];
#pragma unroll
      for (int k = 0; k < MK_KH; ++k) {
        const int i = tid + k * MK_CONSUMERS;
        xv[k] = zv[k] = 0.f;
        if (i < nI) {
          const int c = i % nc, b = i / nc, d = c0 + c;
          xv[k] = __ldcg(p.xzT + (int64_t)d * BP + b);
          zv[k] = __ldcg(p.xzT + (int64_t)(Ek + d) * BP + b);
        }
      }
      {  // 1/rms of every row (reading Q16: weight 1)
        if (l == 0) {  // copy-in partials, fixed order
          float* part = sRed;  // [256 / BP][BP]
          const int b = tid % BP, grp = tid / BP;
          const int ngr = MK_CONSUMERS / BP;
          float a = 0.f;
          for (int c = grp; c < G; c += ngr) a += __ldcg(p.ssP + (int64_t)c * BP + b);
          part[grp * BP + b] = a;
          named_bar_sync(1, MK_CONSUMERS);
          if (tid < BP) {
            float s2 = 0.f;
            for (int j = 0; j < ngr; ++j) s2 += part[j * BP + tid];
            sRS[tid] = tid < B ? rsqrtf(s2 / (float)D + p.eps) : 0.f;
          }
        } else if (tid < BP) {
          sRS[tid] = tid < B ? rsqrtf(__ldcg(p.ss + (e & 1) * BP + tid) / (float)D + p.eps) : 0.f;
        }
        cp_async_wait<1>();  // phase-B/C operands landed (W_dt may still be in flight)
        named_bar_sync(1, MK_CONSUMERS);
        for (int i = tid; i < nc * MK_N; i += MK_CONSUMERS) {
          const int c = i % nc, n = i / nc;
          sA2[n * ncm + c] = -expf(sAl[c * MK_N + n]) * LOG2E;
        }
      }
      if (st0) mk_stamp(p, l, 16);
      auto conv_item = [&](int i, float xraw) {
        const int c = i % nc, b = i / nc, d = c0 + c;
        const float x = bf16r(xraw * sRS[b]);
        const __nv_bfloat16* wsm = sConv + b * (K - 1) * ncm + c;
        float win[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) win[j] = j < K - 1 ? __bfloat162float(wsm[j * ncm]) : 0.f;
        float xc = sCb[c];
        const float* wk = sCw + c * K;
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (j < K - 1) xc = fmaf(wk[j], win[j], xc);
        xc = fmaf(wk[K - 1], x, xc);
        const float uval = bf16r(silu<true>(xc));
        __nv_bfloat16* cwg = Ly.conv + (int64_t)b * (K - 1) * Ek + d;  // the cache window, shifted in place
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (j < K - 2) cwg[(int64_t)j * Ek] = __float2bfloat16_rn(win[j + 1]);
        cwg[(int64_t)(K - 2) * Ek] = __float2bfloat16_rn(x);
        su[b * ncm + c] = uval;
        sub[b * LDX + c] = __float2bfloat16_rn(uval);
        p.xzT[(int64_t)d * BP + b] = 0.f;
      };
#pragma unroll
      for (int k = 0; k < MK_KH; ++k)
        if (tid + k * MK_CONSUMERS < nI) conv_item(tid + k * MK_CONSUMERS, xv[k]);
      for (int i = tid + MK_KH * MK_CONSUMERS; i < nI; i += MK_CONSUMERS)
        conv_item(i, __ldcg(p.xzT + (int64_t)(c0 + i % nc) * BP + i / nc));
      named_bar_sync(1, MK_CONSUMERS);
      if (st0) mk_stamp(p, l, 17);
      float* dbc = p.dbcT + (size_t)(e & 1) * P * BP;
      const uint32_t wx_base = smem_u32(sWx), u_base = smem_u32(sub);
      for (int mt = warp; mt < P / 16; mt += MK_CONSUMERS / 32) {
        float acc[BP / 8][4];
#pragma unroll
        for (int j = 0; j < BP / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        for (int ks = 0; ks < nc / 16; ++ks) {
          uint32_t a[4];
          ldsm_x4(a, wx_base + ((mt * 16 + (m8 & 1) * 8 + r8) * LDX + ks * 16 + (m8 >> 1) * 8) * 2);
#pragma unroll
          for (int jn = 0; jn < BP / 16; ++jn) {
            uint32_t b[4];
            ldsm_x4(b, u_base + ((jn * 16 + (m8 >> 1) * 8 + r8) * LDX + ks * 16 + (m8 & 1) * 8) * 2);
            mma_16816_bf16(acc[2 * jn], a, b[0], b[1]);
            mma_16816_bf16(acc[2 * jn + 1], a, b[2], b[3]);
          }
        }
        const int p0 = mt * 16 + g;
#pragma unroll
        for (int j = 0; j < BP / 8; ++j) {
          const int b = j * 8 + 2 * t;
          if (b < B) {
            red_add_v2(dbc + (int64_t)p0 * BP + b, acc[j][0], acc[j][1]);
            red_add_v2(dbc + (int64_t)(p0 + 8) * BP + b, acc[j][2], acc[j][3]);
          }
        }
      }
    }
    if (st0) mk_stamp(p, l, 4);
    __threadfence();
    mk_grid_sync(p.bar, p.err, t0);  // dbc complete

    // ================= phase C: decode step (a4-a7) for this CTA's channels
    if (nc > 0) {
      if (st0) mk_stamp(p, l, 5);
      const float* dbc = p.dbcT + (size_t)(e & 1) * P * BP;
      for (int q = tid; q < P * BP / 4; q += MK_CONSUMERS)
        reinterpret_cast<float4*>(sD)[q] = __ldcg(reinterpret_cast<const float4*>(dbc) + q);
      named_bar_sync(1, MK_CONSUMERS);
      if (st0) mk_stamp(p, l, 18);
      if (p.rmsnorm) {  // weightless RMSNorm of dt_low, B, C per row (Falcon-Mamba, reading Q18)
        for (int b = warp; b < B; b += MK_CONSUMERS / 32) {
          float s0 = 0.f, s1 = 0.f, s2 = 0.f;
          for (int c = lane; c < P; c += 32) {
            const float v = sD[c * BP + b];
            if (c < R) s0 = fmaf(v, v, s0);
            else if (c < R + MK_N) s1 = fmaf(v, v, s1);
            else s2 = fmaf(v, v, s2);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          }
          if (lane == 0) {
            sNS[b * 3 + 0] = 1.0f / sqrtf(s0 / (float)R + p.rms_eps);
            sNS[b * 3 + 1] = 1.0f / sqrtf(s1 / (float)MK_N + p.rms_eps);
            sNS[b * 3 + 2] = 1.0f / sqrtf(s2 / (float)MK_N + p.rms_eps);
          }
        }
        named_bar_sync(1, MK_CONSUMERS);
      }
      for (int i = tid; i < BP * R; i += MK_CONSUMERS) {  // dt_low as the bf16 B operand [BP][R+8]
        const int b = i % BP, r = i / BP;
        float v = sD[r * BP + b];
        if (p.rmsnorm && b < B) v *= sNS[b * 3 + 0];
        sDl[b * LDR + r] = __float2bfloat16_rn(v);
      }
      cp_async_wait<0>();
      named_bar_sync(1, MK_CONSUMERS);
      if (warp < nc / 16) {  // dt_proj: [nc x R] x [R x BP] on the tensor pipe
        const uint32_t w_base = smem_u32(sWdt), x_base = smem_u32(sDl);
        float acc[BP / 8][4];
#pragma unroll
        for (int j = 0; j < BP / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        for (int ks = 0; ks < R / 16; ++ks) {
          uint32_t a[4];
          ldsm_x4(a, w_base + ((warp * 16 + (m8 & 1) * 8 + r8) * LDR + ks * 16 + (m8 >> 1) * 8) * 2);
#pragma unroll
          for (int jn = 0; jn < BP / 16; ++jn) {
            uint32_t b[4];
            ldsm_x4(b, x_base + ((jn * 16 + (m8 >> 1) * 8 + r8) * LDR + ks * 16 + (m8 & 1) * 8) * 2);
            mma_16816_bf16(acc[2 * jn], a, b[0], b[1]);
            mma_16816_bf16(acc[2 * jn + 1], a, b[2], b[3]);
          }
        }
        const int cc = warp * 16 + g;
#pragma unroll
        for (int j = 0; j < BP / 8; ++j) {
          const int b = j * 8 + 2 * t;
          sdt[b * ncm + cc] = acc[j][0];
          sdt[(b + 1) * ncm + cc] = acc[j][1];
          sdt[b * ncm + cc + 8] = acc[j][2];
          sdt[(b + 1) * ncm + cc + 8] = acc[j][3];
        }
      }
      named_bar_sync(1, MK_CONSUMERS);
      if (st0) mk_stamp(p, l, 19);
      auto scan_item = [&](int i, float zraw, float (&h)[MK_N]) {
        const int c = i % nc, b = i / nc, d = c0 + c;
        const float z = bf16r(zraw * sRS[b]);
        const float dt = softplus(sdt[b * ncm + c] + sBdt[c]);
        const float uu = su[b * ncm + c];
        const float du = dt * uu;
        const float sB = p.rmsnorm ? sNS[b * 3 + 1] : 1.f;
        const float sC = p.rmsnorm ? sNS[b * 3 + 2] : 1.f;
        float y = 0.f;
#pragma unroll
        for (int n = 0; n < MK_N; ++n) {
          const float dA = ex2_approx(dt * sA2[n * ncm + c]);
          h[n] = fmaf(dA, h[n], du * (sD[(R + n) * BP + b] * sB));
          y = fmaf(sD[(R + MK_N + n) * BP + b] * sC, h[n], y);
        }
        float4* hp = reinterpret_cast<float4*>(Ly.h + ((int64_t)b * Ek + d) * MK_N);
#pragma unroll
        for (int n = 0; n < MK_N; n += 4) hp[n / 4] = make_float4(h[n], h[n + 1], h[n + 2], h[n + 3]);
        y = fmaf(sDsk[c], uu, y);
        p.gT[mk_bidx<BP>(d, b)] = __float2bfloat16_rn(y * silu<true>(z));
        p.xzT[(int64_t)(Ek + d) * BP + b] = 0.f;
      };
#pragma unroll
      for (int k = 0; k < MK_KH; ++k)
        if (tid + k * MK_CONSUMERS < nI) scan_item(tid + k * MK_CONSUMERS, zv[k], hs[k]);
      for (int i = tid + MK_KH * MK_CONSUMERS; i < nI; i += MK_CONSUMERS) {
        const int c = i % nc, b = i / nc, d = c0 + c;
        float h[MK_N];
        const float4* hp = reinterpret_cast<const float4*>(Ly.h + ((int64_t)b * Ek + d) * MK_N);
#pragma unroll
        for (int n = 0; n < MK_N; n += 4) {
          const float4 v = __ldcg(hp + n / 4);
          h[n] = v.x; h[n + 1] = v.y; h[n + 2] = v.z; h[n + 3] = v.w;
        }
        scan_item(i, __ldcg(p.xzT + (int64_t)(Ek + d) * BP + b), h);
      }
    }
    if (st0) mk_stamp(p, l, 6);
    fence_proxy_async_global();  // generic writes of g -> bulk-copy (async-proxy) reads
    __threadfence();
    mk_grid_sync(p.bar, p.err, t0);  // g complete
    if (st0) mk_stamp(p, l, 7);

    // ================= phase D: out_proj (a8) + residual add (a9, TP=1) + row-tile finalisation
    const bool last_layer = l + 1 == p.n_layers;
    mk_stage_b<BP>(smem, L, rg, bitc, v0, v1, nkb4, p.gT, p.err, t0, p.dbg);
    if (st0) mk_stamp(p, l, 22);
    mk_epi<BP>(rg, tc, v0, v1, nkb4, p.residT, p.err, t0, [&](int rt) {
      if (!(p.dbg & 8)) __threadfence();  // this thread's partials of residual row tile rt are performed
      named_bar_sync(1, MK_CONSUMERS);
      if (st0) {
        if (p.dbg & 8) __threadfence();
        const uint32_t target = (uint32_t)mk_owners(rt * nkb4, (rt + 1) * nkb4, U4, G) * (e + 1);
        const uint32_t old = atom_add_acq_rel_gpu(cnt + CN.out + 8 * rt, 1u);
        *sFlag = (old + 1u == target);
      }
      named_bar_sync(1, MK_CONSUMERS);
      if (*sFlag) {  // the last contributor: rows [128 rt, 128 rt + 128) are final
        constexpr int Q = 128 * BP / 4;  // float4 of the row tile
        float ssum[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q = tid; q < Q; q += MK_CONSUMERS) {
          const int d = rt * 128 + (q * 4) / BP, b = (q * 4) % BP;
          const float4 v = __ldcg(reinterpret_cast<const float4*>(p.residT + (int64_t)d * BP + b));
          p.residB[mk_bidx<BP>(d, b)] = __float2bfloat16_rn(v.x);
          p.residB[mk_bidx<BP>(d, b + 1)] = __float2bfloat16_rn(v.y);
          p.residB[mk_bidx<BP>(d, b + 2)] = __float2bfloat16_rn(v.z);
          p.residB[mk_bidx<BP>(d, b + 3)] = __float2bfloat16_rn(v.w);
          ssum[0] = fmaf(v.x, v.x, ssum[0]);
          ssum[1] = fmaf(v.y, v.y, ssum[1]);
          ssum[2] = fmaf(v.z, v.z, ssum[2]);
          ssum[3] = fmaf(v.w, v.w, ssum[3]);
          if (last_layer) {
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (b + j < B) p.resid[(int64_t)(b + j) * D + d] = vv[j];
          }
        }
        // thread tid always holds columns 4 (tid % (BP/4)) .. +3: fold threads with equal tid % (BP/4)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          for (int o = BP / 4; o < 32; o <<= 1) ssum[j] += __shfl_xor_sync(0xffffffffu, ssum[j], o);
        if (lane < BP / 4) {
#pragma unroll
          for (int j = 0; j < 4; ++j) sRed[warp * BP + lane * 4 + j] = ssum[j];
        }
        named_bar_sync(1, MK_CONSUMERS);
        if (tid < BP) {
          float a = 0.f;
          for (int w = 0; w < MK_CONSUMERS / 32; ++w) a += sRed[w * BP + tid];
          if (tid < B) atomicAdd(p.ss + ((e + 1) & 1) * BP + tid, a);
        }
      }
    });
    if (st0) mk_stamp(p, l, 8);
    fence_proxy_async_global();  // residB (generic writes) -> next in_proj's bulk copies
    __threadfence();
    mk_grid_sync(p.bar, p.err, t0);  // residual (fp32 + bf16 copy + sums of squares) complete
    if (st0) mk_stamp(p, l, 9);
  }
  if (st0) p.ep[cta] = e0 + p.n_layers;
  tc_fence_before();
  named_bar_sync(2, MK_CONSUMERS + 32);
}

}  // namespace

size_t mk_smem_bytes(int BP, int P, int R, int ncmax, int ring, int nbr) {
  return mk_layout(BP, P, R, ncmax, ring, nbr).total;
}

int mk_ring_slots(int BP, int P, int R, int ncmax, int nbr) {
  constexpr size_t kMax = 227 * 1024 - 1024;  // opt-in limit minus static shared memory headroom
  const size_t base = mk_smem_bytes(BP, P, R, ncmax, 0, nbr);
  if (base >= kMax) return 0;
  int s = (int)((kMax - base) / (MK_TILE + 16));
  while (s > 0 && mk_smem_bytes(BP, P, R, ncmax, s, nbr) > kMax) --s;
  return s > 12 ? 12 : s;
}

cudaError_t launch_decode_mk(const MkParams& p, int BP, int grid, cudaStream_t s) {
  const size_t smem = mk_smem_bytes(BP, p.P, p.R, p.ncmax, p.ring, p.nbr);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(MK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (cross-CTA waits)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (p.dbg & 128) ? 0 : 1;  // experiment: plain launch (1 CTA/SM by shared memory)
  if (BP == 16) return cudaLaunchKernelEx(&cfg, decode_mk_kernel<16>, p);
  if (BP == 32) return cudaLaunchKernelEx(&cfg, decode_mk_kernel<32>, p);
  return cudaErrorInvalidValue;
}

cudaError_t preload_decode_mk() {
  const int smax = 227 * 1024;
  cudaError_t e = cudaFuncSetAttribute(decode_mk_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(decode_mk_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
  return e;
}

}  // namespace ssm
