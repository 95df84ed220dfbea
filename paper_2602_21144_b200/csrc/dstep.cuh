// dstep.cuh — the decode step of one mixer layer for one token per sequence (SURVEY.md §8 a4-a7,
// a10): fixed-order sum of the dbc partials (AR#1 consumer, reading
// Q12) + optional Falcon dt/B/C RMSNorm (Q18), dt_proj + softplus (threshold 20), one ZOH/Euler
// scan step (Q1) with h updated in place, D skip and the SiLU(z) gate.
//
// The work unit is DS_CH channels x DS_BB batch rows, one (b, d) item per thread of a 128-thread
// group, one unit per block of decode_step_kernel (kernels.cu).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace ssm {

constexpr int DS_CH = 32;
constexpr int DS_BB = 4;                       // batch rows per item slot (threads = DS_CH x DS_BB)
constexpr int DS_THREADS = DS_CH * DS_BB;

struct DStepArgs {
  int64_t src_off;       // byte offset of the dbc partials inside each source buffer
  int ldp;               // dbc row stride (floats) = h_loc * P
  int rmsnorm;
  float eps;
  const void* u;         // [batch][Ek]
  const void* z;         // [batch][ldz] (or zacc)
  int64_t ldz;
  const void* w_dt;      // [Ek][R]
  const float* b_dt;
  const float* a_log;    // [Ek][N]
  const float* d_skip;
  float* h;              // [batch][Ek][N] fp32, in place
  void* g;               // [batch][Ek] out
  int batch, Ek, R, cph;
  float* zacc;           // optional fp32 z accumulator (read then zeroed)
};

// W_dt row stride (elements): 16-B aligned, and a 4-word bank shift from row to row (conflict-free LDS.128)
__host__ __device__ inline int dstep_rw(int R, int es) {
  return es == 2 ? R + ((8 - R % 64) + 64) % 64 : R + ((4 - R % 32) + 32) % 32;
}
// shared memory of one unit of DS_BB * IPT batch rows (bytes)
__host__ __device__ inline size_t dstep_smem(int R, int N, int es, int ipt = 1) {
  const int P = R + 2 * N;
  const int RW = dstep_rw(R, es), P4 = (P + 3) & ~3;
  return (size_t)((DS_CH * RW * es + 15) / 16 * 16) +
         (size_t)(DS_BB * ipt * P4 + DS_CH * N + DS_BB * ipt * 3) * sizeof(float);
}
inline bool dstep_supported(int bf16, int R, int N, int ldp, int cph) {
  const int es = bf16 ? 2 : 4;
  return cph % DS_CH == 0 && (N == 16 || N == 8) && dstep_smem(R, N, es, 4) <= 48 * 1024 && (R * es) % 16 == 0 &&
         (R + 2 * N) % 4 == 0 && ldp % 4 == 0;
}

// Synchronise the unit's thread group: whole block (bar_id < 0) or a named barrier of NT threads.
template <int NT>
SSM_DEV void dstep_sync(int bar_id) {
  if (bar_id < 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(NT) : "memory");
}

// One unit: channels [c0, c0 + DS_CH) x batch rows [b0, b0 + DS_BB * IPT); thread tid in [0, NT)
// owns channel c0 + tid % DS_CH and batch rows b0 + tid / DS_CH + DS_BB * i (i < IPT): its IPT
// items share each W_dt register load, and all their global loads are in flight together.
// with_pdl_wait: issue the weight loads, then griddepcontrol.wait before reading activations.
template <typename T, int N, bool FAST, int NT, int IPT>
SSM_DEV void dstep_unit(const DStepArgs& a, const Peers& src, int nsrc, int c0, int b0, int tid, float* dsm,
                        int bar_id, bool with_pdl_wait) {
  static_assert(NT == DS_THREADS, "DS_CH x DS_BB threads per unit");
  constexpr int V = 16 / sizeof(T);
  constexpr int BB = DS_BB * IPT;  // batch rows of the unit
  const int R = a.R, Ek = a.Ek, batch = a.batch;
  const int P = R + 2 * N;
  const int RW = dstep_rw(R, (int)sizeof(T));
  const int P4 = (P + 3) & ~3;
  T* sW = reinterpret_cast<T*>(dsm);                               // [DS_CH][RW] W_dt rows (storage type)
  float* sD = dsm + (DS_CH * RW * (int)sizeof(T) + 15) / 16 * 4;   // [BB][P4] summed dbc rows
  float* sA = sD + BB * P4;                                        // [DS_CH][N] A (log2e-scaled in FAST mode)
  float* sS = sA + DS_CH * N;                                      // [BB][3] RMSNorm scales
  const int hd = c0 / a.cph;
  const int nb = min(BB, batch - b0);
  const T* w_dt = reinterpret_cast<const T*>(a.w_dt);

  // ---- weights first (independent of the predecessor kernels): W_dt rows by cp.async, a_log
  constexpr int AMAX = (DS_CH * N + NT - 1) / NT;
  const int cpr = R / V;
  const int nw = DS_CH * cpr;
  for (int i = tid; i < nw; i += NT) {
    const int c = i / cpr, q = i % cpr;
    const bool okw = c0 + c < Ek;
    cp_async16(sW + c * RW + q * V, w_dt + (int64_t)(okw ? c0 + c : 0) * R + q * V, okw);
  }
  cp_async_commit();
  float al[AMAX];
#pragma unroll
  for (int k = 0; k < AMAX; ++k) {
    const int i = tid + k * NT;
    const int c = i / N, n = i % N;
    al[k] = (i < DS_CH * N && c0 + c < Ek) ? a.a_log[(int64_t)(c0 + c) * N + n] : 0.f;
  }
  const int cc = tid % DS_CH, bl = tid / DS_CH;
  const int d = c0 + cc;
  const bool okd = d < Ek;
  const float bias = okd ? a.b_dt[d] : 0.f;
  const float Dd = okd ? a.d_skip[d] : 0.f;
  // the items' h rows, written by the previous token's decode step: that kernel is only a
  // transitive predecessor (PDL guarantees the completion of the immediate predecessor grid
  // alone, and every kernel of the chain triggers its dependents at entry), so h is read after
  // griddepcontrol.wait, which returns once the whole chain up to this kernel has completed
  if (with_pdl_wait) pdl_wait();  // everything below reads what the predecessor kernels produced
  float hs[IPT][N];
  {
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
      const int bi = bl + DS_BB * it;
      const bool ok = bi < nb && okd;
      const float* hp = a.h + ((int64_t)(ok ? b0 + bi : 0) * Ek + (ok ? d : 0)) * N;
#pragma unroll
      for (int n = 0; n < N; n += 4) {
        const float4 t4 = ok ? *reinterpret_cast<const float4*>(hp + n) : make_float4(0.f, 0.f, 0.f, 0.f);
        hs[it][n] = t4.x; hs[it][n + 1] = t4.y; hs[it][n + 2] = t4.z; hs[it][n + 3] = t4.w;
      }
    }
  }
  // ---- activations: dbc rows (first source), the items' h rows, u, z -- all loads in flight
  const int p4 = P / 4;
  const int nd = nb * p4;
  constexpr int DMAX = 4;
  float4 acc[DMAX];
  const float* sp0 = reinterpret_cast<const float*>(reinterpret_cast<const char*>(src.p[0]) + a.src_off);
  if (nsrc == 1) {  // single source: straight copy into shared memory, no register staging
    for (int i = tid; i < nd; i += NT)
      cp_async16(sD + (i / p4) * P4 + 4 * (i % p4), sp0 + (int64_t)(b0 + i / p4) * a.ldp + (int64_t)hd * P + 4 * (i % p4),
                 true);
    cp_async_commit();
  } else {
#pragma unroll
    for (int k = 0; k < DMAX; ++k) {
      const int i = tid + k * NT;
      acc[k] = i < nd ? *reinterpret_cast<const float4*>(sp0 + (int64_t)(b0 + i / p4) * a.ldp + (int64_t)hd * P + 4 * (i % p4))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  // u and z: every item's loads issued back to back with no branch between them (raw bits; the
  // conversion happens after the shared-memory barrier below), so their latencies overlap each
  // other and the dbc copy instead of adding up
  T ur[IPT], zr[IPT];
  float zz[IPT];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int bi = bl + DS_BB * it;
    const bool ok = bi < nb && okd;
    const int64_t row = ok ? b0 + bi : b0;
    const int dd = okd ? d : c0;
    ur[it] = reinterpret_cast<const T*>(a.u)[row * Ek + dd];
    if (!a.zacc) zr[it] = reinterpret_cast<const T*>(a.z)[row * a.ldz + dd];
  }
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    zz[it] = 0.f;
    const int bi = bl + DS_BB * it;
    if (a.zacc && bi < nb && okd) {
      float* zp = a.zacc + (int64_t)(b0 + bi) * a.ldz + d;
      zz[it] = *zp;
      *zp = 0.f;
    }
  }
  // ---- consume into shared memory; partials of the other sources added in fixed rank order
  for (int base = 0; nsrc > 1 && base < nd; base += DMAX * NT) {
    if (base > 0) {
#pragma unroll
      for (int k = 0; k < DMAX; ++k) {
        const int i = base + tid + k * NT;
        acc[k] = i < nd ? *reinterpret_cast<const float4*>(sp0 + (int64_t)(b0 + i / p4) * a.ldp + (int64_t)hd * P + 4 * (i % p4))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int r = 1; r < kMaxTP; ++r) {  // (compile-time peer index: no local-memory copy of src)
      if (r >= nsrc) break;
      const float* sp = reinterpret_cast<const float*>(reinterpret_cast<const char*>(src.p[r]) + a.src_off);
#pragma unroll
      for (int k = 0; k < DMAX; ++k) {
        const int i = base + tid + k * NT;
        const float4 l4 = i < nd ? *reinterpret_cast<const float4*>(sp + (int64_t)(b0 + i / p4) * a.ldp + (int64_t)hd * P + 4 * (i % p4))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        acc[k].x += l4.x; acc[k].y += l4.y; acc[k].z += l4.z; acc[k].w += l4.w;
      }
    }
#pragma unroll
    for (int k = 0; k < DMAX; ++k) {
      const int i = base + tid + k * NT;
      if (i < nd) *reinterpret_cast<float4*>(sD + (i / p4) * P4 + 4 * (i % p4)) = acc[k];
    }
  }
#pragma unroll
  for (int k = 0; k < AMAX; ++k) {
    const int i = tid + k * NT;
    if (i < DS_CH * N) {
      const float av = -expf(al[k]);
      sA[i] = FAST ? av * 1.4426950408889634f : av;
    }
  }
  cp_async_wait<0>();
  dstep_sync<NT>(bar_id);
  float uu[IPT];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const bool ok = bl + DS_BB * it < nb && okd;
    uu[it] = ok ? io<T>::ld(&ur[it]) : 0.f;
    if (!a.zacc) zz[it] = ok ? io<T>::ld(&zr[it]) : 0.f;
  }
  if (a.rmsnorm) {  // weightless RMSNorm of dt_low, B, C per batch row (Falcon-Mamba, reading Q18)
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = warp; r < nb; r += NT / 32) {
      float s0 = 0.f, s1 = 0.f, s2 = 0.f;
      for (int c = lane; c < P; c += 32) {
        const float v = sD[r * P4 + c];
        if (c < R) s0 = fmaf(v, v, s0);
        else if (c < R + N) s1 = fmaf(v, v, s1);
        else s2 = fmaf(v, v, s2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == 0) {
        sS[r * 3 + 0] = 1.0f / sqrtf(s0 / (float)R + a.eps);
        sS[r * 3 + 1] = 1.0f / sqrtf(s1 / (float)N + a.eps);
        sS[r * 3 + 2] = 1.0f / sqrtf(s2 / (float)N + a.eps);
      }
    }
    dstep_sync<NT>(bar_id);
  }
  if (!okd) return;
  // ---- dt_proj: each W_dt register load serves the thread's IPT batch rows
  const T* wr = sW + cc * RW;
  float sd[IPT][2];
#pragma unroll
  for (int it = 0; it < IPT; ++it) sd[it][0] = sd[it][1] = 0.f;
  for (int r = 0; r < R; r += V) {  // R % V == 0 (dstep_supported)
    float wv[V];
    if constexpr (sizeof(T) == 2) {
      const uint4 raw = *reinterpret_cast<const uint4*>(wr + r);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int j = 0; j < V / 2; ++j) { const float2 f = __bfloat1622float2(b2[j]); wv[2 * j] = f.x; wv[2 * j + 1] = f.y; }
    } else {
      const float4 f = *reinterpret_cast<const float4*>(wr + r);
      wv[0] = f.x; wv[1] = f.y; wv[2] = f.z; wv[3] = f.w;
    }
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
      const float* xr = sD + (bl + DS_BB * it) * P4;
#pragma unroll
      for (int j = 0; j < V; j += 4) {
        const float4 xv = *reinterpret_cast<const float4*>(xr + r + j);
        sd[it][0] = fmaf(xv.x, wv[j], sd[it][0]); sd[it][1] = fmaf(xv.y, wv[j + 1], sd[it][1]);
        sd[it][0] = fmaf(xv.z, wv[j + 2], sd[it][0]); sd[it][1] = fmaf(xv.w, wv[j + 3], sd[it][1]);
      }
    }
  }
  const float* Ac = sA + cc * N;
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int bi = bl + DS_BB * it;
    if (bi >= nb) break;
    const float* xr = sD + bi * P4;
    float dt = sd[it][0] + sd[it][1];
    if (a.rmsnorm) dt *= sS[bi * 3 + 0];
    const float de = softplus(dt + bias);
    const float du = de * uu[it];
    const float sBs = a.rmsnorm ? sS[bi * 3 + 1] : 1.f;
    const float sCs = a.rmsnorm ? sS[bi * 3 + 2] : 1.f;
    const float* Bt = xr + R;
    const float* Ct = xr + R + N;
    float y = 0.f;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float ab = FAST ? ex2_approx(de * Ac[n]) : expf(de * Ac[n]);
      hs[it][n] = fmaf(ab, hs[it][n], du * (Bt[n] * sBs));
      y = fmaf(Ct[n] * sCs, hs[it][n], y);
    }
    float* hp = a.h + ((int64_t)(b0 + bi) * Ek + d) * N;
#pragma unroll
    for (int n = 0; n < N; n += 4)
      *reinterpret_cast<float4*>(hp + n) = make_float4(hs[it][n], hs[it][n + 1], hs[it][n + 2], hs[it][n + 3]);
    y = fmaf(Dd, uu[it], y);
    io<T>::st(reinterpret_cast<T*>(a.g) + (int64_t)(b0 + bi) * Ek + d, y * silu<FAST>(zz[it]));
  }
}

}  // namespace ssm
