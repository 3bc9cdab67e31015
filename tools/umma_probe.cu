// tcgen05.mma issue-rate probe: clocks per MMA for kind::tf32 / kind::f16
// at M=128 and N in {64, 128, 256}, A from shared memory or TMEM.  One CTA,
// operands are zeros (timing only).  Diagnostic only; build: tools/build_tools.sh.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {  // K-major SWIZZLE_128B, SBO 1024
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, bool kF16, bool kTA, int kNoise = 0>
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tmem_sh;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_sh)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_sh;
  if (kNoise && threadIdx.x >= 32) {
    // background shared-memory traffic (kNoise = 1: reads, 2: reads + writes)
    // over a separate 32 KiB region while warp 0 issues MMAs
    volatile int* flag = reinterpret_cast<volatile int*>(out + 1);
    const uint32_t base = su32(smem + 65536);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < 20000 && *flag == 0; ++it) {
      const uint32_t a = base + (uint32_t)(((threadIdx.x - 32) * 16 + it * 1536) & 32767);
      float4 v;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
      acc.x += v.x;
      if (kNoise == 2)
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a ^ 16384u), "f"(acc.x), "f"(v.y), "f"(v.z),
                     "f"(v.w));
    }
    if (acc.x == 12345.f) out[2] = 1;
  }
  if (threadIdx.x == 0) {
    // idesc: D f32 (bit 4), A/B kind (tf32: 2 at bits 7 and 10; f16 family bf16: 1), K-major, N>>3 at 17, M>>4 at 24
    const uint32_t ab = kF16 ? 1u : 2u;
    const uint32_t idesc = (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t da = kdesc(su32(smem)), db = kdesc(su32(smem + 32768));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (kTA) {
        if (kF16)
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(tmem + 256u),
                       "l"(db), "r"(idesc));
        else
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(tmem + 256u),
                       "l"(db), "r"(idesc));
      } else {
        if (kF16)
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da), "l"(db),
                       "r"(idesc));
        else
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da), "l"(db),
                       "r"(idesc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            su32(&bar))
        : "memory");
    out[0] = clock64() - t0;
    *reinterpret_cast<volatile int*>(out + 1) = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, bool kF16, bool kTA, int kNoise = 0>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 32);
  cudaMemset(d, 0, 32);
  const int smem = 97 * 1024 + 32768;
  cudaFuncSetAttribute(probe<N, kF16, kTA, kNoise>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  probe<N, kF16, kTA, kNoise><<<1, kNoise ? 512 : 128, smem>>>(d, iters);
  cudaMemset(d + 1, 0, 8);
  probe<N, kF16, kTA, kNoise><<<1, kNoise ? 512 : 128, smem>>>(d, iters);
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / iters;
  const double k = kF16 ? 16 : 8;
  printf("%-26s N=%3d  %7.1f clk/MMA  %7.0f FLOP/clk/SM  (%s)\n", name, N, per, 2.0 * 128 * N * k / per,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, false, false>("tf32 A smem");
  run<128, false, false>("tf32 A smem");
  run<256, false, false>("tf32 A smem");
  run<64, false, true>("tf32 A tmem");
  run<128, false, true>("tf32 A tmem");
  run<256, false, true>("tf32 A tmem");
  run<128, true, false>("bf16 A smem");
  run<256, true, false>("bf16 A smem");
  run<256, true, true>("bf16 A tmem");
  run<128, false, false, 1>("tf32 A smem + 15 warps lds");
  run<128, false, false, 2>("tf32 A smem + lds/sts");
  run<128, false, true, 1>("tf32 A tmem + 15 warps lds");
  run<128, false, true, 2>("tf32 A tmem + lds/sts");
  return 0;
}
