// Throughput probe: legacy mma.sync m16n8k8 tf32 (HMMA) on sm_100a, 8 warps
// per CTA, independent accumulator chains.  Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(float* out, int iters, long long* cyc) {
  float c[4][4] = {};
  unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  unsigned b[2] = {threadIdx.x * 3u, threadIdx.x * 5u};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int warps : {1, 4, 8}) {
    const int iters = 4096;
    probe<<<148, 32 * warps>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    const double mma_per_sm = 4.0 * iters * warps;
    printf("warps/CTA %d: %.2f cycles per mma.sync (per SM), %.0f FLOP/clk/SM tf32\n", warps, h[0] / mma_per_sm,
           mma_per_sm * 16 * 8 * 8 * 2 / h[0]);
  }
  return 0;
}
