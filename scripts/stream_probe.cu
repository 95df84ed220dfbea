// Read-bandwidth probe (experiment tool, not part of libssmtp): how fast can ONE kernel launch
// stream a decode-sized weight matrix (26-52 MB) from HBM on B200?  Two read engines:
//   ldg : grid-stride LDG.128 with UNROLL independent loads in flight per thread
//   bulk: one elected thread per CTA drives a ring of cp.async.bulk (TMA 1D) copies into smem
// Built and driven by scripts/stream_probe.py.
#include <cstdint>
#include <cuda_runtime.h>

extern "C" __global__ void __launch_bounds__(512) ldg_stream(const int4* __restrict__ p, long long n16,
                                                             int* __restrict__ sink) {
    constexpr int U = 8;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    int acc = 0;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        int4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
    unsigned a = (unsigned)__cvta_generic_to_shared(b);
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(a), "r"(ph));
}

// ring of S stages x CH bytes per CTA; each CTA streams a contiguous slice
extern "C" __global__ void bulk_stream(const char* __restrict__ p, long long bytes, int S, int CH, int* sink) {
    extern __shared__ __align__(128) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    char* ring = smem + 1024;
    const long long per = (bytes / gridDim.x) & ~15LL;
    const char* src = p + per * blockIdx.x;
    const int nch = (int)((per + CH - 1) / CH);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int c = 0; c < nch + S; ++c) {
        if (c >= S) {  // retire chunk c - S
            int s = (c - S) % S;
            mbar_wait(bar + s, ((c - S) / S) & 1);
        }
        if (c < nch) {
            int s = c % S;
            unsigned len = (unsigned)min((long long)CH, per - (long long)c * CH);
            mbar_expect(bar + s, len);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    (unsigned)__cvta_generic_to_shared(ring + (size_t)s * CH)),
                "l"(src + (long long)c * CH), "r"(len), "r"((unsigned)__cvta_generic_to_shared(bar + s))
                : "memory");
        }
    }
    if (ring[0] == 123 && ring[1] == 45) sink[0] = 1;
}

extern "C" int probe_ldg(const void* p, long long bytes, int grid, int block, int* sink, cudaStream_t s) {
    ldg_stream<<<grid, block, 0, s>>>((const int4*)p, bytes / 16, sink);
    return (int)cudaGetLastError();
}

extern "C" int probe_bulk(const void* p, long long bytes, int grid, int S, int CH, int* sink, cudaStream_t s) {
    int sm = 1024 + S * CH;
    cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    bulk_stream<<<grid, 32, sm, s>>>((const char*)p, bytes, S, CH, sink);
    return (int)cudaGetLastError();
}
