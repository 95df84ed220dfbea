// probe_cluster_coop.cu — can the persistent decode kernel's launch (148 CTAs x 512 threads, ~220 KB
// dynamic smem, cooperative) also carry a 2-CTA cluster dimension on this B200?  Reports
// cudaOccupancyMaxActiveClusters and the launch result, and checks a DSMEM store + remote mbarrier-free
// handshake (barrier.cluster) inside the cooperative grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_cc scripts/probe_cluster_coop.cu && ./probe_cc
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) k_cc(int* out) {
  extern __shared__ int sm[];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) sm[0] = -1;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    // write blockIdx into the partner's sm[0]
    unsigned local = (unsigned)__cvta_generic_to_shared(sm), remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank ^ 1u));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"((unsigned)blockIdx.x) : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 220 * 1024;
  cudaFuncSetAttribute(k_cc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms & ~1);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclu = -1;
  cudaError_t eo = cudaOccupancyMaxActiveClusters(&nclu, (void*)k_cc, &cfg);
  printf("SMs %d, max active 2-CTA clusters at %zu KB smem: %d (%s)\n", sms, smem / 1024, nclu, cudaGetErrorString(eo));
  int* out;
  cudaMalloc(&out, sms * 4);
  cudaMemset(out, 0xff, sms * 4);
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_cc, out);
  cudaError_t e2 = cudaDeviceSynchronize();
  int h[256];
  cudaMemcpy(h, out, sms * 4, cudaMemcpyDeviceToHost);
  int ok = 1;
  for (int i = 0; i < (sms & ~1); ++i) ok &= (h[i] == (i ^ 1));
  printf("cooperative + cluster launch of %d CTAs: launch %s, sync %s, DSMEM exchange %s\n", sms & ~1,
         cudaGetErrorString(e), cudaGetErrorString(e2), ok ? "ok" : "WRONG");
  return 0;
}
