// Tensor-core (tcgen05, sm_100a) GEMM for the wide affine contractions
// (output layer forward / dX / dW and the aggregated recurrent dW):
//
//   C[M x N] (= | +=) A(m,k) B(k,n) (+ bias_m(n))       fp32 in, fp32 out
//
// fp32 parity (rtol 1e-4 against the CPU reference) is kept with 3xTF32:
// the tensor core reads an fp32 operand as TF32 (x_hi), a second operand copy
// holds the residual x_lo = x - x_hi, and the fp32 TMEM accumulator receives
// A_hi*B_hi + A_hi*B_lo + A_lo*B_hi  (3.5e-7 normwise vs fp64).
//
// Pipeline (one 128x128 output tile per CTA, 256 threads, 1 CTA/SM):
//   * cp.async 16-byte chunks (works on gathered row-pointer operands) bring
//     raw fp32 k-tiles (128 x 32) of A and B into a 4-stage ring, already in
//     the UMMA canonical SWIZZLE_128B layout -- K-major when the operand's
//     rows run along M/N, MN-major when they run along K (no transposes);
//   * the raw tile is the "hi" MMA operand; all threads write the residual
//     "lo" tile (a layout-agnostic elementwise pass, double-buffered);
//   * thread 0 issues 12 tcgen05.mma.kind::tf32 (M=128, N=128, K=8) per
//     k-tile and commits to a per-stage mbarrier that releases the raw stage
//     and the lo buffer;
//   * epilogue: tcgen05.ld 32x32b from TMEM, bias / accumulate, stores.
//   * split-K: the splits of one tile form a thread-block cluster; partials
//     are reduced through distributed shared memory in split order
//     (deterministic; no global partials, no atomics).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace cgrp = cooperative_groups;

namespace dg {
namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32;
constexpr int kTcThreads = 256;
constexpr int kTileBytes = 128 * TBK * 4;  // 16 KiB: 128 (M or N) x 32 (K) fp32
constexpr int kRawStages = 4;
constexpr int kLoStages = 2;
constexpr int kSmemBytes = (kRawStages * 2 + kLoStages * 2) * kTileBytes + 1024;

__device__ __forceinline__ const float* op_row(const Operand& o, int64_t i) {
  return o.rows ? o.rows[i] : o.base + i * o.ld;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, version 1 (sm_100).
//   K-major : SWIZZLE_128B (layout 2): rows of 128 B (32 K), 8-row groups
//             1024 B apart (SBO); LBO unused
//   MN-major: SWIZZLE_128B_BASE32B (layout 1, the only MN-major layout for
//             tf32): 4-row x 128 B atoms, 4-row K groups 512 B apart (SBO),
//             32-element MN groups 4096 B apart (LBO)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, bool mn_major) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((mn_major ? (4096 >> 4) : 1) & 0x3FFF) << 16;
  d |= (uint64_t)(((mn_major ? 512 : 1024) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(mn_major ? 1 : 2) << 61;
  return d;
}

// instruction descriptor: D f32, A/B tf32, N=128, M=128, operand majors
__host__ __device__ constexpr uint32_t umma_idesc(bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((TBN >> 3) << 17) | ((TBM >> 4) << 24);
}

// byte offset of 16-byte chunk c of tile row r (K-major: r = M/N index, c =
// k/4) or of K row r, MN chunk c (MN-major), inside one 16 KiB tile
__device__ __forceinline__ uint32_t off_kmajor(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }
// MN-major (Swizzle<2,5,2>): 32-byte chunk index XOR (K row % 4)
__device__ __forceinline__ uint32_t off_mnmajor(int k, int c) {
  const int g = c >> 3, c16 = c & 7, kk = k & 3, kg = k >> 2;
  return (uint32_t)(g * 4096 + kg * 512 + kk * 128 + ((((c16 >> 1) ^ kk) << 5) | ((c16 & 1) << 4)));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issue the cp.async of one 128 x 32 operand tile.
//   kRowK == false: global rows run along M/N (K contiguous) -> K-major smem
//   kRowK == true : global rows run along K (M/N contiguous) -> MN-major smem
template <bool kRowK>
__device__ __forceinline__ void load_tile(uint32_t dst, const Operand& op, const float* const* rowcache, bool vec,
                                          int64_t mn0, int64_t mn_lim, int64_t k0, int64_t k_lim,
                                          const void* dummy) {  // any valid global address (zero-fill source)
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = tid + i * kTcThreads;  // 1024 chunks of 16 B
    if (!kRowK) {
      const int r = idx >> 3, c = idx & 7;  // row r, k chunk c
      const int64_t gr = mn0 + r, gk = k0 + 4 * c;
      const uint32_t d = dst + off_kmajor(r, c);
      const float* row = gr < mn_lim ? rowcache[r] : nullptr;
      const int64_t rem = k_lim - gk;
      const int valid = row ? (rem >= 4 ? 4 : (rem > 0 ? (int)rem : 0)) : 0;
      if (vec) {
        cp_async16(d, valid ? (const void*)(row + gk) : dummy, valid * 4);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) cp_async4(d + 4 * q, q < valid ? (const void*)(row + gk + q) : dummy, q < valid ? 4 : 0);
      }
    } else {
      const int k = idx >> 5, c = idx & 31;  // k row, MN chunk c
      const int64_t gk = k0 + k, gm = mn0 + 4 * c;
      const uint32_t d = dst + off_mnmajor(k, c);
      const float* row = gk < k_lim ? op_row(op, gk) : nullptr;
      const int64_t rem = mn_lim - gm;
      const int valid = row ? (rem >= 4 ? 4 : (rem > 0 ? (int)rem : 0)) : 0;
      if (vec) {
        cp_async16(d, valid ? (const void*)(row + gm) : dummy, valid * 4);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) cp_async4(d + 4 * q, q < valid ? (const void*)(row + gm + q) : dummy, q < valid ? 4 : 0);
      }
    }
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// residual lo = x - tf32(x) (the tensor core reads fp32 storage as TF32 by
// dropping the low 13 mantissa bits)
__device__ __forceinline__ float tf32_lo(float x) { return tf32_rn_lo_of_raw(x); }

// kAMN: A global rows run along K (MN-major A); kBMN: B global rows run along K
// TMEM accumulator -> registers: 64 fp32 columns of this thread's row
__device__ __forceinline__ void tmem_drain_add(uint32_t tmem, int lane_grp, int col_half, float* vals) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    const uint32_t taddr = tmem + ((uint32_t)(lane_grp * 32) << 16) + (uint32_t)(col_half * 64 + c * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 32; ++q) vals[c * 32 + q] += __uint_as_float(r[q]);
  }
}

// chunk: drain the TMEM accumulator into fp32 registers every `chunk` k-tiles
// (blocked summation: the tensor core's own accumulation error grows with the
// chain length, see tools/gemm_bench.cu accuracy study)
template <bool kAMN, bool kBMN>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_kernel(const GemmProblem* __restrict__ probs, int n_probs, int chunk) {
  pdl_prologue();
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // ring: raw[s] = {A 16K, B 16K}, lo[b] = {A 16K, B 16K}
  char* raw = smem;
  char* lo = smem + kRawStages * 2 * kTileBytes;
  __shared__ uint64_t bars[kRawStages];
  __shared__ uint32_t tmem_base_sh;
  __shared__ GemmProblem P;
  __shared__ const float* rowA[kAMN ? 1 : TBM];
  __shared__ const float* rowB[kBMN ? 1 : TBN];

  int p = 0;
  while (p + 1 < n_probs && (int)blockIdx.x >= __ldg(&probs[p + 1].cta0)) ++p;
  {
    const int* src = reinterpret_cast<const int*>(probs + p);
    int* dst = reinterpret_cast<int*>(&P);
    for (int i = threadIdx.x; i < (int)(sizeof(GemmProblem) / 4); i += blockDim.x) dst[i] = src[i];
  }
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRawStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  const int local = blockIdx.x - P.cta0;
  const int S = P.splits;
  const int z = local % S, tile = local / S;
  const int64_t m0 = (int64_t)(tile / P.tiles_n) * TBM, n0 = (int64_t)(tile % P.tiles_n) * TBN;
  if (!kAMN)
    for (int i = threadIdx.x; i < TBM; i += blockDim.x) rowA[i] = m0 + i < P.M ? op_row(P.seg[0].A, m0 + i) : nullptr;
  if (!kBMN)
    for (int i = threadIdx.x; i < TBN; i += blockDim.x) rowB[i] = n0 + i < P.N ? op_row(P.seg[0].B, n0 + i) : nullptr;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  const int kt_total = (int)((P.seg[0].K + TBK - 1) / TBK);
  const int t0 = (int)((int64_t)kt_total * z / S), t1 = (int)((int64_t)kt_total * (z + 1) / S);
  const int nkt = t1 - t0;
  const GemmSeg& sg = P.seg[0];
  const bool va = P.vec_a, vb = P.vec_b;
  const uint32_t raw_u = smem_u32(raw), lo_u = smem_u32(lo);
  auto issue = [&](int j) {  // cp.async k-tile t0+j into raw stage j % 4
    if (j < nkt) {
      const int64_t k0 = (int64_t)(t0 + j) * TBK;
      const uint32_t dA = raw_u + (j % kRawStages) * 2 * kTileBytes;
      load_tile<kAMN>(dA, sg.A, rowA, va, m0, P.M, k0, sg.K, probs);
      load_tile<kBMN>(dA + kTileBytes, sg.B, rowB, vb, n0, P.N, k0, sg.K, probs);
    }
    cp_async_commit();  // one (possibly empty) group per stage keeps the wait counts uniform
  };
  constexpr uint32_t idesc = umma_idesc(kAMN, kBMN);
  const int lane_grp = warp & 3, col_half = warp >> 2;
  const int lrow = lane_grp * 32 + (threadIdx.x & 31);
  float vals[64];
#pragma unroll
  for (int q = 0; q < 64; ++q) vals[q] = 0.f;
#pragma unroll
  for (int j = 0; j < kRawStages - 1; ++j) issue(j);
  for (int j = 0; j < nkt; ++j) {
    const int s = j % kRawStages, b = j % kLoStages;
    // raw stage s of tile j has landed (this thread's copies), then everyone's
    cp_async_wait<kRawStages - 2>();
    __syncthreads();
    // the lo buffer b was last read by the MMAs of tile j-2: wait for them
    if (j >= kLoStages) mbar_wait(&bars[(j - kLoStages) % kRawStages], ((j - kLoStages) / kRawStages) & 1);
    // residual pass: raw[s] -> lo[b] (same layout, elementwise)
    {
      const float4* src = reinterpret_cast<const float4*>(raw + s * 2 * kTileBytes);
      float4* dst = reinterpret_cast<float4*>(lo + b * 2 * kTileBytes);
#pragma unroll
      for (int i = 0; i < (2 * kTileBytes / 16) / kTcThreads; ++i) {
        const int e = threadIdx.x + i * kTcThreads;
        float4 x = src[e];
        dst[e] = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = raw_u + s * 2 * kTileBytes, b_hi = a_hi + kTileBytes;
      const uint32_t a_lo = lo_u + b * 2 * kTileBytes, b_lo = a_lo + kTileBytes;
#pragma unroll
      for (int ks = 0; ks < TBK / 8; ++ks) {
        // K-major: 8 tf32 = 32 B along the 128 B row; MN-major: next 8-row K group
        const uint32_t oa = kAMN ? ks * 1024 : ks * 32, ob = kBMN ? ks * 1024 : ks * 32;
        const uint32_t first = (j % chunk == 0 && ks == 0) ? 0u : 1u;
        mma_tf32(tmem, umma_desc(a_hi + oa, kAMN), umma_desc(b_hi + ob, kBMN), idesc, first);
        mma_tf32(tmem, umma_desc(a_hi + oa, kAMN), umma_desc(b_lo + ob, kBMN), idesc, 1u);
        mma_tf32(tmem, umma_desc(a_lo + oa, kAMN), umma_desc(b_hi + ob, kBMN), idesc, 1u);
      }
      mma_commit(&bars[s]);
    }
    // chunk boundary: wait for this tile's MMAs, fold the accumulator into
    // fp32 registers; the next chunk restarts the TMEM accumulation
    if ((j + 1) % chunk == 0 || j + 1 == nkt) {
      mbar_wait(&bars[s], (j / kRawStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      tmem_drain_add(tmem, lane_grp, col_half, vals);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // every warp drained before the next scale_c = 0 MMA
    }
    // refill: tile j+3 goes to raw stage (j+3)%4, last read by the MMAs of tile j-1
    if (j + kRawStages - 1 < nkt && j >= 1) mbar_wait(&bars[(j - 1) % kRawStages], ((j - 1) / kRawStages) & 1);
    issue(j + kRawStages - 1);
  }
  cp_async_wait<0>();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();  // all TMEM reads done; the operand ring is free
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TBN));

  const bool has_bias = P.bias.rows != nullptr || P.bias.base != nullptr;
  if (S > 1) {
    float* part = reinterpret_cast<float*>(smem);  // 128 x 128 fp32 = 64 KiB
#pragma unroll
    for (int q = 0; q < 64; q += 4)
      *reinterpret_cast<float4*>(part + lrow * TBN + col_half * 64 + q) =
          make_float4(vals[q], vals[q + 1], vals[q + 2], vals[q + 3]);
    cgrp::cluster_group cl = cgrp::this_cluster();
    cl.sync();
    const int rows = TBM / S;  // S is a power of two <= 8
    for (int e = threadIdx.x; e < rows * (TBN / 4); e += blockDim.x) {
      const int lm = z * rows + e / (TBN / 4), ln = (e % (TBN / 4)) * 4;
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < S; ++q) {
        const float4 x = *reinterpret_cast<const float4*>(cl.map_shared_rank(part, q) + lm * TBN + ln);
        s4.x += x.x;
        s4.y += x.y;
        s4.z += x.z;
        s4.w += x.w;
      }
      const int64_t m = m0 + lm;
      if (m < P.M) {
        float* crow = const_cast<float*>(op_row(P.C, m));
        const float* brow = has_bias ? op_row(P.bias, m) : nullptr;
        const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t n = n0 + ln + q;
          if (n < P.N) {
            float v = sv[q];
            if (brow) v += brow[n];
            if (P.accumulate) v += crow[n];
            crow[n] = v;
          }
        }
      }
    }
    cl.sync();
    return;
  }
  const int64_t m = m0 + lrow;
  if (m < P.M) {
    float* crow = const_cast<float*>(op_row(P.C, m));
    const float* brow = has_bias ? op_row(P.bias, m) : nullptr;
#pragma unroll
    for (int q = 0; q < 64; ++q) {
      const int64_t n = n0 + col_half * 64 + q;
      if (n < P.N) {
        float v = vals[q];
        if (brow) v += brow[n];
        if (P.accumulate) v += crow[n];
        crow[n] = v;
      }
    }
  }
}

template <bool kAMN, bool kBMN>
void launch_tc(const GemmLaunch& L, const GemmProblem* probs, cudaStream_t s) {
  auto kern = tc_gemm_kernel<kAMN, kBMN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L.ctas);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = L.cluster > 0 ? L.cluster : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, probs, L.n_probs, L.chunk > 0 ? L.chunk : 1 << 30);
}

bool vec_ok(const Operand& o, int64_t extent) {
  if (extent % 4) return false;
  if (o.rows) return o.rows_aligned != 0;
  return (reinterpret_cast<uintptr_t>(o.base) % 16 == 0) && (o.ld % 4 == 0);
}

}  // namespace

bool tc_gemm_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Tensor-core eligibility: single-segment problems with every dimension wide
// enough to fill 128 x 128 tiles.
bool tc_gemm_eligible(const std::vector<GemmProblem>& probs) {
  if (!tc_gemm_enabled()) return false;
  for (const auto& p : probs) {
    if (p.n_seg != 1) return false;
    if (p.M < 128 || p.N < 128 || p.seg[0].K < 256) return false;  // short K: the SIMT kernel wins
  }
  return !probs.empty();
}

// a_kmajor (A(m,k) = A.row(k)[m]) => MN-major A in shared memory; b_nmajor
// (B(k,n) = B.row(n)[k]) => K-major B, otherwise MN-major B.
GemmLaunch tc_gemm_plan(std::vector<GemmProblem>& probs, bool a_kmajor, bool b_nmajor) {
  GemmLaunch L{};
  L.cfg = 10;  // tensor-core path
  L.a_kmajor = a_kmajor;
  L.b_nmajor = b_nmajor;
  L.n_probs = (int)probs.size();
  int64_t tiles_all = 0;
  int min_kt = 1 << 30;
  for (auto& p : probs) {
    p.tiles_n = (p.N + TBN - 1) / TBN;
    p.tiles = ((p.M + TBM - 1) / TBM) * p.tiles_n;
    tiles_all += p.tiles;
    min_kt = std::min<int>(min_kt, (int)((p.seg[0].K + TBK - 1) / TBK));
  }
  // split-K (a cluster of S CTAs per tile) until ~one wave of 148 SMs
  int S = 1;
  while (S < 8 && tiles_all * S * 2 <= 148 && min_kt >= 8 * S) S *= 2;
  L.cluster = S;
  // TMEM drain period (k-tiles of 32): DG_TC_CHUNK overrides (accuracy studies)
  static const int chunk_env = [] {
    const char* e = getenv("DG_TC_CHUNK");
    return e ? atoi(e) : 0;
  }();
  L.chunk = chunk_env > 0 ? chunk_env : 2;
  int64_t cta = 0;
  for (auto& p : probs) {
    p.splits = S;
    p.cta0 = (int)cta;
    cta += (int64_t)p.tiles * S;
    p.vec_a = vec_ok(p.seg[0].A, a_kmajor ? p.M : p.seg[0].K);
    p.vec_b = vec_ok(p.seg[0].B, b_nmajor ? p.seg[0].K : p.N);
    L.flops += 2.0 * p.M * p.N * (double)p.seg[0].K;
  }
  L.ctas = (int)cta;
  return L;
}

int launch_tc_gemm(const GemmLaunch& L, const GemmProblem* probs_dev, cudaStream_t s) {
  if (L.ctas <= 0) return 0;
  // global rows along K: A when a_kmajor, B when !b_nmajor
  if (L.a_kmajor && !L.b_nmajor) launch_tc<true, true>(L, probs_dev, s);
  else if (L.a_kmajor) launch_tc<true, false>(L, probs_dev, s);
  else if (!L.b_nmajor) launch_tc<false, true>(L, probs_dev, s);
  else launch_tc<false, false>(L, probs_dev, s);
  return 1;
}

}  // namespace dg
