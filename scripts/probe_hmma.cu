// probe_hmma.cu — mma.sync.m16n8k16 bf16 (HMMA) latency and throughput on one B200 SM:
// W warps x C independent accumulator chains x N mma each, timed with clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_hmma scripts/probe_hmma.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k(long long* out, int n, unsigned a0) {
  float acc[C][4];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
  unsigned a[4] = {a0, a0 + 1, a0 + 2, a0 + 3}, b0 = a0 ^ 5, b1 = a0 ^ 9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][3];
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (s == 1234.5f) out[1] = 1;
}

template <int C>
void run(int warps) {
  long long* d;
  cudaMalloc(&d, 16);
  const int n = 2000;
  k<C><<<1, 32 * warps>>>(d, n, 7);
  k<C><<<1, 32 * warps>>>(d, n, 7);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / n / C;  // cycles per mma per warp-chain step
  printf("warps %2d chains %d: %.1f cycles per mma per warp; SM throughput %.2f mma/cycle\n", warps, C, per * 1.0,
         (double)warps * C * n / h);
  cudaFree(d);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<1>(w);
    run<4>(w);
  }
  return 0;
}
