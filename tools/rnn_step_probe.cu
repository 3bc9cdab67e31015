// Recurrence-step A/B probe: clocks for ONE step's recurrent contraction of
// the persistent LSTM kernels (rnn.cu), G[gate cols x rows] += W h^T over
// K = 256 in 3xTF32, as
//   (a) legacy mma.sync m16n8k8 (the shipped rnn_fwd_cl_kernel loop: 8 warps,
//       64 gate columns x 16 rows, 96 MMAs per warp), result to smem + barrier;
//   (b) tcgen05.mma kind::tf32, one thread issues 3 x 32 MMAs of 128 x N x 8
//       (128 gate columns = 32 units, N = batch rows), commit -> mbarrier,
//       4 warps tcgen05.ld the accumulator, barrier.
// Operands are zeros (timing only).  One CTA.  Diagnostic only:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/rnn_step_probe.cu -o tools/rnn_step_probe
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
__device__ __forceinline__ void mma_1688(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }
__device__ __forceinline__ uint32_t tf32_lo(float x) {
  return __float_as_uint(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
}

// (a) the shipped loop; kMode 1: operands from registers (HMMA throughput
// only), 2: shared-memory loads only (no HMMA), 3: A pre-split {hi, lo}
// pairs (LDS.64, no ALU split)
template <int kMode = 0>
__global__ void __launch_bounds__(256, 1) step_mma_sync(long long* out, int iters) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int KS = 32, HP = 8 * KS + 4;
  float4* Bf = sm4;
  float* hS = sm + KS * 8 * 32 * 4;
  float* gS = hS + 2 * 16 * HP;
  for (int i = threadIdx.x; i < KS * 8 * 32 * 4 + 2 * 16 * HP + 16 * 68; i += 256) sm[i] = 0.f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float* r0 = hS + g8 * (kMode == 3 ? 2 * HP : HP);
    const float* r1 = hS + (g8 + 8) * (kMode == 3 ? 2 * HP : HP);
    float ac[6][4];
#pragma unroll
    for (int z = 0; z < 6; ++z) ac[z][0] = ac[z][1] = ac[z][2] = ac[z][3] = 0.f;
    const float4* bw = Bf + warp * 32 + lane;
    float sinkv = 0.f;
    if (kMode == 4) {
      // warp w: n-tiles 2(w%4), 2(w%4)+1 over k-steps [16 (w/4), +16)
      const float4* bw0 = Bf + (2 * (warp & 3)) * 32 + lane;
      const float4* bw1 = bw0 + 32;
      float ad[6][4];
#pragma unroll
      for (int z = 0; z < 6; ++z) ad[z][0] = ad[z][1] = ad[z][2] = ad[z][3] = 0.f;
      const int q0 = 16 * (warp >> 2);
#pragma unroll 4
      for (int q = q0; q < q0 + 16; ++q) {
        const int k = 8 * q + t4;
        float av[4] = {r0[k], r1[k], r0[k + 4], r1[k + 4]};
        uint32_t ah[4], al[4];
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          ah[z] = tf32_hi(av[z]);
          al[z] = tf32_lo(av[z]);
        }
        const float4 b = bw0[q * 256], c = bw1[q * 256];
        mma_1688(ac[0], al, __float_as_uint(b.x), __float_as_uint(b.y));
        mma_1688(ac[1], ah, __float_as_uint(b.z), __float_as_uint(b.w));
        mma_1688(ac[2], ah, __float_as_uint(b.x), __float_as_uint(b.y));
        mma_1688(ad[0], al, __float_as_uint(c.x), __float_as_uint(c.y));
        mma_1688(ad[1], ah, __float_as_uint(c.z), __float_as_uint(c.w));
        mma_1688(ad[2], ah, __float_as_uint(c.x), __float_as_uint(c.y));
      }
      ac[3][0] += ad[0][0] + ad[1][1] + ad[2][2];
    } else
#pragma unroll 4
    for (int q = 0; q < KS; ++q) {
      const int k = 8 * q + t4;
      uint32_t ah[4], al[4];
      float4 b;
      if (kMode == 1) {
        b = make_float4(__int_as_float(q), 0.f, 0.f, 0.f);
#pragma unroll
        for (int z = 0; z < 4; ++z) ah[z] = al[z] = (uint32_t)(q + z);
      } else if (kMode == 3) {
        const float2* x0 = reinterpret_cast<const float2*>(r0);
        const float2* x1 = reinterpret_cast<const float2*>(r1);
        const float2 p0 = x0[k], p1 = x1[k], p2 = x0[k + 4], p3 = x1[k + 4];
        b = bw[q * 256];
        ah[0] = __float_as_uint(p0.x); ah[1] = __float_as_uint(p1.x); ah[2] = __float_as_uint(p2.x); ah[3] = __float_as_uint(p3.x);
        al[0] = __float_as_uint(p0.y); al[1] = __float_as_uint(p1.y); al[2] = __float_as_uint(p2.y); al[3] = __float_as_uint(p3.y);
      } else {
        float av[4] = {r0[k], r1[k], r0[k + 4], r1[k + 4]};
        b = bw[q * 256];
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          ah[z] = tf32_hi(av[z]);
          al[z] = tf32_lo(av[z]);
        }
      }
      float* c3 = ac[(q & 1) * 3];
      if (kMode == 2) {
        sinkv += b.x + b.y + b.z + b.w + __uint_as_float(ah[0] ^ al[1] ^ ah[2] ^ al[3] ^ ah[1] ^ al[0] ^ ah[3] ^ al[2]);
        continue;
      }
      mma_1688(c3, al, __float_as_uint(b.x), __float_as_uint(b.y));
      mma_1688(c3 + 4, ah, __float_as_uint(b.z), __float_as_uint(b.w));
      mma_1688(c3 + 8, ah, __float_as_uint(b.x), __float_as_uint(b.y));
    }
    ac[0][0] += sinkv;
    float* o0 = gS + g8 * 68 + 8 * warp + 2 * t4;
    *reinterpret_cast<float2*>(o0) = make_float2(ac[0][0] + ac[3][0] + ac[1][0], ac[4][1] + ac[2][1] + ac[5][1]);
    *reinterpret_cast<float2*>(o0 + 8 * 68) = make_float2(ac[0][2] + ac[3][2] + ac[1][2], ac[4][3] + ac[2][3] + ac[5][3]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = clock64() - t0;
}

// (b) tcgen05: NMMA MMAs of 128 x N x 8 per step (3 per k-step, 32 k-steps)
template <int N, bool kTA, int NMMA, int M = 128, bool kHoist = false>
__global__ void __launch_bounds__(256, 1) step_umma(long long* out, int iters) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tmem_sh;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
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
  const int warp = threadIdx.x >> 5;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  const uint64_t da0 = kdesc(su32(smem)), db0 = kdesc(su32(smem + 131072));
  float sink = 0.f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (kHoist) {
#pragma unroll 8
        for (int i = 0; i < NMMA; ++i) {
          if (kTA)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 480u),
                "r"(tmem), "l"(db0), "r"(idesc), "r"(i));
          else
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 480u),
                "l"(da0), "l"(db0), "r"(idesc), "r"(i));
        }
      }
      for (int i = 0; i < (kHoist ? 0 : NMMA); ++i) {
        const uint64_t db = kdesc(su32(smem + 131072 + (i & 31) * 32));
        if (kTA) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 480u),
              "r"(tmem + (uint32_t)((i & 31) * 8)), "l"(db), "r"(idesc), "r"(i));
        } else {
          const uint64_t da = kdesc(su32(smem + (i & 31) * 4096));
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 480u),
              "l"(da), "l"(db), "r"(idesc), "r"(i));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
            su32(&bar)),
        "r"(it & 1)
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
      uint32_t v[N];
      if constexpr (N == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + 480u + ((uint32_t)(warp * 32) << 16)));
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + 480u + ((uint32_t)(warp * 32) << 16)));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < N; ++i) sink += __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = clock64() - t0;
  if (sink == 1234.5f) out[1] = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <class K>
void run(K k, const char* name, int smem, double flop_per_step) {
  long long* d;
  cudaMalloc(&d, 32);
  cudaMemset(d, 0, 32);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k<<<1, 256, smem>>>(d, iters);
  k<<<1, 256, smem>>>(d, iters);
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / iters;
  printf("%-44s %8.1f clk/step  %6.2f us/step @1.965GHz  %7.0f useful FLOP/clk  (%s)\n", name, per, per / 1965.0,
         flop_per_step / per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  const double f64 = 2.0 * 64 * 16 * 256, f128 = 2.0 * 128 * 16 * 256;
  const int sm_ms = 4 * (32 * 8 * 32 * 4 + 2 * 16 * 520 + 16 * 68);
  run(step_mma_sync<0>, "mma.sync 64 cols x 16 rows (shipped)", sm_ms, f64);
  run(step_mma_sync<1>, "mma.sync, operands in registers", sm_ms, f64);
  run(step_mma_sync<2>, "mma.sync loop, smem loads only", sm_ms, f64);
  run(step_mma_sync<3>, "mma.sync, A pre-split pairs (LDS.64)", sm_ms, f64);
  run(step_mma_sync<4>, "mma.sync, K split over warp pairs, 2 n-tiles", sm_ms, f64);
  run(step_umma<16, false, 96>, "tcgen05 128 x 16, A smem, 96 MMA", 161 * 1024 + 2048, f128);
  run(step_umma<16, true, 96>, "tcgen05 128 x 16, A tmem, 96 MMA", 161 * 1024 + 2048, f128);
  run(step_umma<8, false, 96>, "tcgen05 128 x 8, A smem, 96 MMA", 161 * 1024 + 2048, f128 / 2);
  run(step_umma<8, true, 96>, "tcgen05 128 x 8, A tmem, 96 MMA", 161 * 1024 + 2048, f128 / 2);
  run(step_umma<16, false, 1>, "tcgen05 128 x 16, 1 MMA (round trip)", 161 * 1024 + 2048, 0);
  run(step_umma<16, true, 64>, "tcgen05 128 x 16, A tmem, 64 MMA", 161 * 1024 + 2048, f128);
  run(step_umma<16, false, 96, 128, true>, "hoisted 128 x 16, A smem, 96 MMA", 161 * 1024 + 2048, f128);
  run(step_umma<16, true, 96, 128, true>, "hoisted 128 x 16, A tmem, 96 MMA", 161 * 1024 + 2048, f128);
  run(step_umma<64, false, 96, 128, true>, "hoisted 128 x 64, A smem, 96 MMA", 161 * 1024 + 2048, 4 * f128);
  run(step_umma<128, false, 96, 128, true>, "hoisted 128 x 128, A smem, 96 MMA", 161 * 1024 + 2048, 8 * f128);
  run(step_umma<16, false, 96, 64, true>, "hoisted 64 x 16, A smem, 96 MMA", 161 * 1024 + 2048, f128 / 2);
  run(step_umma<16, true, 96, 64, true>, "hoisted 64 x 16, A tmem, 96 MMA", 161 * 1024 + 2048, f128 / 2);
  return 0;
}
