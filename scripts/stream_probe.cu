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

// Burst probe: each CTA issues `n` bulk copies of `ch` bytes (all in flight at once, one mbarrier),
// waits for all, `reps` times.  Time per burst tells whether TMA bulk copies overlap.
extern "C" __global__ void bulk_burst(const char* __restrict__ p, long long span, int n, int ch, int reps,
                                      int issuers, int* sink) {
    extern __shared__ __align__(128) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    char* buf = smem + 1024;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const char* src = p + ((long long)blockIdx.x * n * ch) % (span - (long long)n * ch);
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x == 0) mbar_expect(bar, (unsigned)(n * ch));
        __syncwarp();
        if (threadIdx.x < issuers) {
            for (int i = threadIdx.x; i < n; i += issuers)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        (unsigned)__cvta_generic_to_shared(buf + (size_t)i * ch)),
                    "l"(src + (long long)i * ch), "r"(ch), "r"((unsigned)__cvta_generic_to_shared(bar))
                    : "memory");
        }
        if (threadIdx.x == 0) mbar_wait(bar, r & 1);
        __syncwarp();
    }
    if (buf[0] == 123 && buf[1] == 45) sink[0] = 1;
}

extern "C" int probe_burst(const void* p, long long span, int grid, int n, int ch, int reps, int issuers, int* sink,
                           cudaStream_t s) {
    int sm = 1024 + n * ch;
    cudaFuncSetAttribute(bulk_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    bulk_burst<<<grid, 32, sm, s>>>((const char*)p, span, n, ch, reps, issuers, sink);
    return (int)cudaGetLastError();
}

// mbarrier try_wait cost on an already-completed phase (cycles per call), and elect/syncwarp cost
extern "C" __global__ void mbar_cost(long long* out, int iters) {
    __shared__ uint64_t bar[4];
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned a = (unsigned)__cvta_generic_to_shared(bar);
        long long t0 = clock64();
        unsigned okc = 0;
        for (int i = 0; i < iters; ++i) {
            unsigned ok;
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(a), "r"(0u) : "memory");
            okc += ok;
        }
        long long t1 = clock64();
        for (int i = 0; i < iters; ++i) {
            unsigned ok;
            asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(a), "r"(0u) : "memory");
            okc += ok;
        }
        long long t2 = clock64();
        unsigned long long g0, g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        for (int i = 0; i < iters; ++i) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        }
        long long t3 = clock64();
        out[0] = (t1 - t0) / iters;
        out[1] = (t2 - t1) / iters;
        out[2] = (t3 - t2) / iters;
        out[3] = okc;
    }
}
extern "C" int probe_mbar(long long* out, int iters, cudaStream_t s) {
    mbar_cost<<<1, 32, 0, s>>>(out, iters);
    return (int)cudaGetLastError();
}

// Does an mbarrier last arrived by tcgen05.commit cost more to probe than one arrived by a thread?
extern "C" __global__ void commit_probe(long long* out, int mode) {
    __shared__ __align__(8) uint64_t bar[32];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 32; ++i) mbar_init(bar + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((unsigned)__cvta_generic_to_shared(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x == 32) {
        for (int i = 0; i < 22; ++i) {
            unsigned a = (unsigned)__cvta_generic_to_shared(bar + i);
            if (mode == 1)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a) : "memory");
            else
                asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(a) : "memory");
        }
    }
    // wait (thread 0) until the last one completed, then time 22 probes of completed phases
    if (threadIdx.x == 0) {
        unsigned a = (unsigned)__cvta_generic_to_shared(bar + 21);
        unsigned ok = 0;
        while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a) : "memory");
        long long t0 = clock64();
        unsigned c = 0;
        for (int i = 0; i < 22; ++i) {
            unsigned a2 = (unsigned)__cvta_generic_to_shared(bar + i);
            asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a2) : "memory");
            c += ok;
        }
        long long t1 = clock64();
        for (int i = 0; i < 22; ++i) {
            unsigned a2 = (unsigned)__cvta_generic_to_shared(bar + i);
            asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a2) : "memory");
            c += ok;
        }
        long long t2 = clock64();
        out[mode * 4 + 0] = t1 - t0;
        out[mode * 4 + 1] = t2 - t1;
        out[mode * 4 + 2] = c;
    }
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
    }
}
extern "C" int probe_commit(long long* out, cudaStream_t s) {
    commit_probe<<<1, 128, 0, s>>>(out, 0);
    commit_probe<<<1, 128, 0, s>>>(out, 1);
    return (int)cudaGetLastError();
}
