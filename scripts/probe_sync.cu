// probe_sync.cu — microbenchmarks for the persistent decode's latency floors on one B200:
//   (1) grid barrier (bar.sync + red.release + acquire poll) over 148 CTAs x 480 threads
//   (2) one L2 round trip after a barrier: every CTA reads the SAME 12 KB (broadcast, like the x_proj
//       sums) vs its OWN 12 KB, by 480 threads with 16-B cp.async, timed with clock64 on thread 0
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_sync scripts/probe_sync.cu && ./probe_sync
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void bar1(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_vol(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// variant 0: red.release + ld.acquire poll; 1: red.release + relaxed poll + fence.acquire;
// 2: fence + red.relaxed + volatile poll + fence; 3: variant 1 without the CTA bar.syncs (thread 0 only)
__device__ int g_variant;
__device__ unsigned g_flags[160 * 32];  // one 128-B line per CTA
__device__ __forceinline__ void gsync(unsigned* bar, unsigned target, int nthr) {
  const int v = g_variant;
  if (v == 9 || v == 10) {
    // 9: no fences at all (latency floor; not a correct barrier); 10: relaxed arrive + relaxed poll,
    // one fence.acq_rel before the arrive and one after the poll
    bar1(nthr);
    if (threadIdx.x == 0) {
      if (v == 10) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
      while (ld_rlx(bar) < target) {
      }
      if (v == 10) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    bar1(nthr);
    return;
  }
  if (v >= 6) {
    // arrivals spread over K counters (one 128-B line each); a warp polls all K and sums
    const int K = v == 6 ? 8 : (v == 7 ? 16 : 32);
    const unsigned per = target / gridDim.x;  // barrier index
    bar1(nthr);
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(g_flags + (blockIdx.x % K) * 32) : "memory");
      while (true) {
        unsigned c = threadIdx.x < K ? ld_acq(g_flags + threadIdx.x * 32) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (c >= per * gridDim.x) break;
      }
    }
    bar1(nthr);
    return;
  }
  if (v >= 4) {
    // last arriver (atom.add returns the old count) writes the generation into every CTA's own flag
    // line; each CTA polls only its line (no 148-way hot spot)
    bar1(nthr);
    if (threadIdx.x < 32) {
      unsigned old = 0;
      if (threadIdx.x == 0) {
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
      }
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old == target - 1) {
        for (int c = threadIdx.x; c < gridDim.x; c += 32)
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(g_flags + c * 32), "r"(target) : "memory");
      }
      if (threadIdx.x == 0) {
        if (v == 4) {
          while (ld_acq(g_flags + blockIdx.x * 32) < target) {
          }
        } else {
          while (ld_rlx(g_flags + blockIdx.x * 32) < target) {
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
      }
    }
    bar1(nthr);
    return;
  }
  if (v != 3) bar1(nthr);
  if (threadIdx.x == 0) {
    if (v == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
      while (ld_acq(bar) < target) {
      }
    } else if (v == 1 || v == 3) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
      while (ld_rlx(bar) < target) {
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    } else {
      __threadfence();
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
      while (ld_vol(bar) < target) {
      }
      __threadfence();
    }
  }
  if (v != 3) bar1(nthr);
}

__global__ void k_probe(unsigned* bar, const float4* buf, long long* out, int iters, int mode) {
  __shared__ float4 sm[768];
  const int nc = gridDim.x, nthr = blockDim.x;
  unsigned nb = 0;
  long long tb = 0, tl = 0;
  for (int it = 0; it < iters; ++it) {
    long long t0 = clock64();
    gsync(bar, (++nb) * nc, nthr);
    long long t1 = clock64();
    // one round trip: 12 KB per CTA by cp.async (mode 0: broadcast, 1: distinct per CTA)
    const float4* src = buf + (mode ? (size_t)blockIdx.x * 768 : 0);
    for (int i = threadIdx.x; i < 768; i += nthr) {
      unsigned s = (unsigned)__cvta_generic_to_shared(&sm[i]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(src + i) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    bar1(nthr);
    long long t2 = clock64();
    if (it > 2) { tb += t1 - t0; tl += t2 - t1; }
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = tb / (iters - 3);
    out[2 * blockIdx.x + 1] = tl / (iters - 3);
  }
  if (sm[threadIdx.x % 768].x == 12345.f) out[0] = 0;  // keep the loads
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* bar;
  float4* buf;
  long long* out;
  cudaMalloc(&bar, 4);
  cudaMalloc(&buf, (size_t)sms * 768 * 16);
  cudaMalloc(&out, (size_t)sms * 16);
  cudaMemset(buf, 0, (size_t)sms * 768 * 16);
  for (int var = 0; var < 11; ++var)
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemcpyToSymbol(g_variant, &var, 4);
    cudaMemset(bar, 0, 4);
    {
      void* fp;
      cudaGetSymbolAddress(&fp, g_flags);
      cudaMemset(fp, 0, sizeof(unsigned) * 160 * 32);
    }
    void* args[] = {&bar, &buf, &out, nullptr, &mode};
    int iters = 200;
    args[3] = &iters;
    cudaLaunchCooperativeKernel((void*)k_probe, sms, 480, args, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2 * 160];
    cudaMemcpy(h, out, (size_t)sms * 16, cudaMemcpyDeviceToHost);
    double sb = 0, sl = 0;
    long long mb = 0, ml = 0;
    for (int i = 0; i < sms; ++i) {
      sb += h[2 * i]; sl += h[2 * i + 1];
      if (h[2 * i] > mb) mb = h[2 * i];
      if (h[2 * i + 1] > ml) ml = h[2 * i + 1];
    }
    const double ghz = clk / 1e6;
    printf("variant %d %s (%s): grid barrier mean %.0f cyc (%.2f us), max %.0f;  12 KB cp.async round trip mean %.0f cyc (%.2f us), max %lld\n",
           var, mode ? "distinct" : "broadcast", cudaGetErrorString(e), sb / sms, sb / sms / ghz / 1e3, (double)mb, sl / sms,
           sl / sms / ghz / 1e3, ml);
  }
  return 0;
}
