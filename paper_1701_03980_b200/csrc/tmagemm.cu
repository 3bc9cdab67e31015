// Warp-specialised tcgen05 3xTF32 GEMM with TMA operand loads (sm_100a) for
// the wide affine contractions whose operands are dense row-major blocks in
// the arena (the output layer of a batched RNNLM: logits = H W^T + b,
// dH = dLogits W, dW^T += H^T dLogits):
//
//   C[M x N] (= | +=) A(m,k) B(k,n) (+ bias(n))         fp32 in, fp32 out
//
// fp32 parity is kept with 3xTF32: the tensor core reads fp32 storage as TF32
// (x_hi = x with the low 13 mantissa bits dropped); a residual copy
// x_lo = rn(x - x_hi) of each operand is produced once per launch by
// split_lo_kernel into the workspace (or per tile by converter warps; an
// operand split by the converters is rounded to nearest in both parts,
// kernels.cuh tf32_rn_*), and every k-step issues
// A_hi*B_hi + A_hi*B_lo + A_lo*B_hi into an fp32 TMEM accumulator.
// Every CHUNK k-tiles the accumulator is handed to the epilogue warps, which
// add it into fp32 registers (blocked summation: the tensor core's own
// accumulation is not a full-precision fp32 chain over K = 10^4), while the
// MMA warp continues in the second TMEM accumulator.
//
// Roles (192 threads, one CTA per SM, 128 x 128 output tile):
//   warp 0  TMA producer: per k-tile 4 tensor loads (A_hi, A_lo, B_hi, B_lo)
//           into a 3-stage ring (64 KiB per stage) signalling an mbarrier
//           with the transaction byte count;
//   warp 1  TMEM allocation + single-thread tcgen05.mma issue (12 MMAs of
//           128x128x8 per k-tile), tcgen05.commit releases the stage and,
//           at chunk ends, publishes the accumulator;
//   warps 2-5  epilogue: tcgen05.ld drains (each warp its 32-lane TMEM
//           quadrant), bias / accumulate, stores; split-K tiles reduce their
//           partials through distributed shared memory of the cluster, or
//           (when the clusters could not all be co-resident) through a
//           workspace summed in split order by the tile's last CTA.
// Default variants: converter warps (320 threads) form the residuals in
// shared memory / A's split in TMEM; *lite* (K per split <= 1024) runs two
// CTAs per SM with one accumulator.  tma_gemm_pers_kernel below is the
// persistent form (one CTA per SM over tiles or K-split units, double-
// buffered TMEM accumulators, TMA tensor stores of C or of split partials).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "kernels.cuh"

namespace cgrp = cooperative_groups;

namespace dg {
namespace {

constexpr int BM = 128, BN = 128, BK = 32;
constexpr int kStages = 3;
constexpr int kOpBytes = 128 * BK * 4;         // 16 KiB per operand tile
constexpr int kStageBytes = 4 * kOpBytes;      // A_hi, A_lo, B_hi, B_lo
constexpr int kThreads = 192;      // producer, MMA, 4 epilogue warps
constexpr int kThreadsConv = 320;  // + 4 converter warps forming the residuals in shared memory
constexpr int kSmem = kStages * kStageBytes + 1024;
// conversion variant: 5 raw stages (A_hi, B_hi) + 2 residual buffers (A_lo, B_lo)
constexpr int kRawStagesC = 3;
constexpr int kSmemConv = kRawStagesC * 4 * kOpBytes + 1024;
constexpr int kChunk = 4;  // k-tiles per TMEM accumulation (K = 128)
// A-in-TMEM variant: stages of A_raw | B_raw | B_lo (48 KiB) in shared memory;
// the converter warps write A's hi/lo split straight into TMEM (columns
// 256 + 64 s .. +63), so the MMAs read only B from shared memory
constexpr int kStagesAT = 4;
constexpr int kSmemAT = kStagesAT * 3 * kOpBytes + 1024;
// "lite" variant (K per split <= kLiteMaxK): 2 stages, one TMEM
// accumulator over the whole K drained once, 256 TMEM columns and ~97 KiB of
// shared memory, so two CTAs share an SM and one's epilogue overlaps the
// other's mainloop
constexpr int kStagesLite = 2;
constexpr int kSmemLite = kStagesLite * 3 * kOpBytes + 1024;
constexpr int kLiteMaxK = 1024;
// persistent variant: 4 stages of A_raw | B_raw | B_lo, two 16 KiB output
// staging buffers (32 columns each); TMEM: two 128-column accumulators + A's
// hi/lo per stage
constexpr int kStagesPers = 4;
constexpr int kThreadsPers = 448;  // producer, MMA, 4 epilogue, 4 A-converter, 4 B-converter warps
constexpr int kSmemPers = kStagesPers * 3 * kOpBytes + 2 * BM * 32 * 4 + 1024;
constexpr int kLiteMaxKSplit = 768;  // per split, when a cluster reduces the splits

// DG_TMA_DBG bit 10: CTA 0 records (before, after) clock64 of each role's
// per-k-tile wait (diagnostics; tools/tma_bench)
__device__ long long g_tprof[6][256][2];

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra W_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

// UMMA smem descriptors (same layouts as tcgemm.cu): K-major SWIZZLE_128B
// (SBO 1024 B) / MN-major SWIZZLE_128B_BASE32B (LBO 4096 B, SBO 512 B)
__device__ __forceinline__ uint64_t udesc(uint32_t saddr, bool mn) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((mn ? (4096 >> 4) : 1) & 0x3FFF) << 16;
  d |= (uint64_t)(((mn ? 512 : 1024) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(mn ? 1 : 2) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t uidesc(bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((BN >> 3) << 17) | ((BM >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem, uint32_t ta, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
      "r"(ta), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float tf32_lo(float x) { return tf32_rn_lo_of_raw(x); }
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

__device__ __forceinline__ const float* orow(const Operand& o, int64_t i) {
  return o.rows ? o.rows[i] : o.base + i * o.ld;
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// ragged-N / unaligned tiles: element-wise stores (rare; kept out of line)
__device__ __noinline__ void epilogue_scalar(const TmaGemmArgs& P, float* part, const float* gws,
                                             cgrp::cluster_group& cl, int S, int z, int rows, int m0, int n0,
                                             bool has_bias) {
  for (int e = threadIdx.x; e < rows * BN; e += blockDim.x) {
    const int lr = e / BN, c = e % BN;
    const int lm = z * rows + lr;
    const int64_t m = m0 + lm, n = n0 + c;
    if (m >= P.M || n >= P.N) continue;
    const int sw = (c & ~3) + 4 * lm;
    float v = 0.f;
    const int off = lm * BN + (sw & (BN - 1)) + (c & 3);
    for (int q = 0; q < S; ++q)
      v += gws ? __ldcg(gws + (size_t)q * (BM * BN) + off) : (S > 1 ? cl.map_shared_rank(part, q) : part)[off];
    float* crow = const_cast<float*>(orow(P.C, m));
    if (has_bias) v += orow(P.bias, m)[n];
    if (P.accumulate) v += crow[n];
    crow[n] = v;
  }
}

// One launch runs up to kTmaGroup independent problems of the same operand
// majors and split factor (problem i owns CTAs [cta0_i, cta0_{i+1})): the
// small LSTM weight-gradient GEMMs of one backward share a wave instead of
// each under-filling the device.
template <bool kAMN, bool kBMN, bool kConv, bool kAT = false, bool kLite = false>
__global__ void __launch_bounds__(kConv ? kThreadsConv : kThreads, kLite ? 2 : 1)
    tma_gemm_kernel(const __grid_constant__ TmaGroup G) {
  // (pdl_prologue after barrier init / TMEM allocation / descriptor prefetch)
  int pi = 0;
  while (pi + 1 < G.n && (int)blockIdx.x >= G.p[pi + 1].cta0) ++pi;
  const TmaProb& PR = G.p[pi];
  const CUtensorMap& mAh = PR.mAh;
  const CUtensorMap& mAl = PR.mAl;
  const CUtensorMap& mBh = PR.mBh;
  const CUtensorMap& mBl = PR.mBl;
  const TmaGemmArgs& P = PR.args;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  static_assert(!kAT || kConv, "A in TMEM needs the converter warps");
  static_assert(!kLite || kAT, "the lite variant keeps A in TMEM");
  constexpr int NS = kLite ? kStagesLite : kAT ? kStagesAT : kConv ? kRawStagesC : kStages;  // raw operand stages
  // stage stride: A_hi, B_hi, A_lo, B_lo (conv) / A_hi, A_lo, B_hi, B_lo / A, B, B_lo (A in TMEM)
  constexpr int SB = kAT ? 3 * kOpBytes : kStageBytes;
  constexpr uint32_t kTmemCols = kLite ? 256 : kAT ? 512 : 2 * BN;
  constexpr uint32_t kAcol = kLite ? BN : 2 * BN;  // first TMEM column of A's per-stage hi/lo (A in TMEM)
  __shared__ uint64_t full[NS], empty[NS], conv[NS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#define WAITB0(b, ph) mbar_wait(b, ph)
  const bool prof = (P.pad_ & 1024) && blockIdx.x == 0;
#define WAITP(role, jj, b, ph)                                             \
  do {                                                                     \
    const long long tb_ = prof ? clock64() : 0;                            \
    WAITB0(b, ph);                                                         \
    if (prof && (jj) < 256) {                                              \
      g_tprof[role][jj][0] = tb_;                                          \
      g_tprof[role][jj][1] = clock64();                                    \
    }                                                                      \
  } while (0)
  const int S = P.splits;
  const bool prof_e = prof && threadIdx.x == 64;
  if (prof_e) g_tprof[5][0][0] = clock64();
  const int local = (int)blockIdx.x - PR.cta0;
  const int z = local % S, tile = local / S;
  // m-tiles fastest: CTAs that run together share the same B columns, so a
  // streamed B operand (dlogits in dW) is read from DRAM once
  const int tiles_m = (P.M + BM - 1) / BM;
  const int m0 = (tile % tiles_m) * BM, n0 = (tile / tiles_m) * BN;
  const int kt_total = (P.K + BK - 1) / BK;
  const int t0 = (int)((int64_t)kt_total * z / S), t1 = (int)((int64_t)kt_total * (z + 1) / S);
  const int nkt = t1 - t0;
  const int nchunks = (nkt + kChunk - 1) / kChunk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NS; ++b) mbar_init(&conv[b], 4);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAh)) : "memory");
    if (!kConv) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAl)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBh)) : "memory");
    if (!kConv) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBl)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_sh)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // operands / C of the preceding grid are read only from here on (nowait:
  // launched behind an independent grid whose own inputs were complete)
  if (P.nowait) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  else pdl_prologue();
  const uint32_t tmem = tmem_sh;
  const uint32_t sbase = su32(smem);

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < nkt; ++j) {
        const int s = j % NS, use = j / NS;
        if (use > 0) WAITP(0, j, &empty[s], (use - 1) & 1);
        if (P.pad_ & 16) {  // DG_TMA_DBG bit 4: no loads
          mbar_arrive(&full[s]);
          continue;
        }
        mbar_expect_tx(&full[s], kConv ? 2 * kOpBytes : kStageBytes);
        const uint32_t st = sbase + s * SB;
        const int k0 = (t0 + j) * BK;
        // A: K-major box {32 k, 128 m} at (k0, m0); MN-major 4 boxes {32 m, 32 k} at (m0 + 32g, k0)
        if (!kAMN) {
          tma_2d(st, &mAh, k0, m0, &full[s]);
          if (!kConv) tma_2d(st + kOpBytes, &mAl, k0, m0, &full[s]);
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            tma_2d(st + g * 4096, &mAh, m0 + 32 * g, k0, &full[s]);
            if (!kConv) tma_2d(st + kOpBytes + g * 4096, &mAl, m0 + 32 * g, k0, &full[s]);
          }
        }
        const uint32_t sbh = st + (kConv ? kOpBytes : 2 * kOpBytes);
        if (!kBMN) {
          tma_2d(sbh, &mBh, k0, n0, &full[s]);
          if (!kConv) tma_2d(st + 3 * kOpBytes, &mBl, k0, n0, &full[s]);
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            tma_2d(sbh + g * 4096, &mBh, n0 + 32 * g, k0, &full[s]);
            if (!kConv) tma_2d(st + 3 * kOpBytes + g * 4096, &mBl, n0 + 32 * g, k0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = uidesc(kAMN && !kAT, kBMN);
      for (int j = 0; j < nkt; ++j) {
        const int s = j % NS, use = j / NS;
        const int c = kLite ? 0 : j / kChunk, a = c & 1;
        if (!kLite && j % kChunk == 0 && c >= 2) WAITP(1, j, &acc_empty[a], ((c >> 1) - 1) & 1);
        if (kConv) WAITP(2, j, &conv[s], use & 1);
        else WAITP(2, j, &full[s], use & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t ah, al, bh, bl;
        if (kAT) {
          ah = tmem + kAcol + 64u * (uint32_t)s;  // TMEM columns: hi, then lo at +32
          al = ah + 32u;
          bh = sbase + s * SB + kOpBytes;
          bl = bh + kOpBytes;
        } else if (kConv) {
          ah = sbase + s * SB;
          bh = ah + kOpBytes;
          al = ah + 2 * kOpBytes;
          bl = ah + 3 * kOpBytes;
        } else {
          ah = sbase + s * SB;
          al = ah + kOpBytes;
          bh = ah + 2 * kOpBytes;
          bl = ah + 3 * kOpBytes;
        }
        const uint32_t acc = tmem + (uint32_t)(a * BN);
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint32_t oa = kAMN ? ks * 1024 : ks * 32, ob = kBMN ? ks * 1024 : ks * 32;
          const uint32_t first = ((kLite ? j == 0 : j % kChunk == 0) && ks == 0) ? 0u : 1u;
          if (P.pad_ & 1) continue;  // DG_TMA_DBG bit 0: no MMAs (pipeline timing only)
          if (kAT) {
            mma_tf32_ta(acc, ah + 8u * ks, udesc(bh + ob, kBMN), idesc, first);
            mma_tf32_ta(acc, ah + 8u * ks, udesc(bl + ob, kBMN), idesc, 1u);
            mma_tf32_ta(acc, al + 8u * ks, udesc(bh + ob, kBMN), idesc, 1u);
            continue;
          }
          mma_tf32(acc, udesc(ah + oa, kAMN), udesc(bh + ob, kBMN), idesc, first);
          mma_tf32(acc, udesc(ah + oa, kAMN), udesc(bl + ob, kBMN), idesc, 1u);
          mma_tf32(acc, udesc(al + oa, kAMN), udesc(bh + ob, kBMN), idesc, 1u);
        }
        if (P.pad_ & 64) {  // DG_TMA_DBG bit 6 (with bit 0): plain arrives instead of commits
          mbar_arrive(&empty[s]);
          if (j % kChunk == kChunk - 1 || j == nkt - 1) mbar_arrive(&acc_full[a]);
          continue;
        }
        mma_commit(&empty[s]);
        if ((!kLite && j % kChunk == kChunk - 1) || j == nkt - 1) mma_commit(&acc_full[a]);
      }
    }
  } else if (kAT && warp >= 6) {
    // converter warps 6..9 (TMEM lane quadrant q = warp % 4): B's residual
    // into shared memory (elementwise, same swizzled layout) and A row
    // m = 32 q + lane split into hi / lo and stored into TMEM (lane m,
    // 32 columns each), then published to the tensor pipe
    const int ct = threadIdx.x - 6 * 32;  // 0..127
    const int q = warp & 3, m = 32 * q + lane;
    for (int j = 0; j < nkt; ++j) {
      const int s = j % NS, use = j / NS;
      if (ct == 0) WAITP(3, j, &full[s], use & 1);
      else WAITB0(&full[s], use & 1);
      const uint32_t st = sbase + s * SB;
      if (!(P.pad_ & 2)) {
#pragma unroll
        for (int i = 0; i < kOpBytes / 16 / 128; ++i) {
          const uint32_t off = (uint32_t)(ct + i * 128) * 16u;
          const float4 x = lds128(st + kOpBytes + off);
          sts128(st + 2 * kOpBytes + off, make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w)));
        }
        uint32_t hi[32], lo[32];
        if (!kAMN) {  // K-major SW128: row m is one 128 B line, 16 B chunk c at (c ^ (m & 7))
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = lds128(st + (uint32_t)m * 128u + ((uint32_t)(c ^ (m & 7)) << 4));
            const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              hi[4 * c + e] = tf32_rn_bits(xv[e]);
              lo[4 * c + e] = __float_as_uint(xv[e] - __uint_as_float(hi[4 * c + e]));
            }
          }
        } else {  // MN-major box q {32 m, 32 k}, SW128 with 32 B atoms: chunk (lane / 8) ^ (k & 3)
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x = lds32(st + (uint32_t)q * 4096u + (uint32_t)k * 128u +
                                  ((uint32_t)(((lane >> 3) ^ (k & 3))) << 5) + ((uint32_t)(lane & 7) << 2));
            hi[k] = tf32_rn_bits(x);
            lo[k] = __float_as_uint(x - __uint_as_float(hi[k]));
          }
        }
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + kAcol + 64u * (uint32_t)s;
        tmem_st32(ta, hi);
        tmem_st32(ta + 32u, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
    // the epilogue reuses the operand stages for its staging tile: order our
    // last shared-memory reads before its writes explicitly (the mbarrier /
    // tcgen05.commit chain already does; named barrier 2 makes it visible to
    // compute-sanitizer racecheck too)
    asm volatile("bar.arrive 2, 256;" ::: "memory");
  } else if (kConv && warp >= 6) {
    // converter warps 6..9: residual lo = x - tf32(x) of the landed hi tiles
    // (same swizzled layout, elementwise), then publish to the async proxy
    const int ct = threadIdx.x - 6 * 32;  // 0..127
    for (int j = 0; j < nkt; ++j) {
      const int s = j % NS, use = j / NS;
      if (ct == 0) WAITP(3, j, &full[s], use & 1);
      else WAITB0(&full[s], use & 1);
      char* st = smem + s * SB;
      char* lo = st + 2 * kOpBytes;
#pragma unroll
      for (int op = 0; op < 2 && !(P.pad_ & 2); ++op) {  // DG_TMA_DBG bit 1: no conversion
        const float4* src = reinterpret_cast<const float4*>(st + op * kOpBytes);
        float4* dst = reinterpret_cast<float4*>(lo + op * kOpBytes);
#pragma unroll
        for (int i = 0; i < kOpBytes / 16 / 128; ++i) {
          const float4 x = src[ct + i * 128];
          float4 y;
          y.x = tf32_rn_lo_of_raw(x.x);
          y.y = tf32_rn_lo_of_raw(x.y);
          y.z = tf32_rn_lo_of_raw(x.z);
          y.w = tf32_rn_lo_of_raw(x.w);
          dst[ct + i * 128] = y;
        }
      }
      if (!(P.pad_ & 128)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // bit 7: no fence
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
    asm volatile("bar.arrive 2, 256;" ::: "memory");  // see the A-in-TMEM converters
  } else if (kLite) {
    // epilogue warps 2..5: one drain of the whole-K accumulator, 32 columns at
    // a time, straight into the staging tile (no register-resident row)
    const int quad = warp & 3;
    mbar_wait(&acc_full[0], 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("bar.sync 2, 256;" ::: "memory");  // converters done with the stages (kLite implies kConv)
    float* part = reinterpret_cast<float*>(smem);
    const int lrow = quad * 32 + lane;
#pragma unroll 1
    for (int h = 0; h < BN / 32; ++h) {
      uint32_t r[32];
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(h * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
            "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
            "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
            "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; q += 4)
        *reinterpret_cast<float4*>(part + lrow * BN + ((h * 32 + q + 4 * lrow) & (BN - 1))) =
            make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]), __uint_as_float(r[q + 2]),
                        __uint_as_float(r[q + 3]));
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrant warp % 4
    const int quad = warp & 3;
    float vals[BN];  // this thread's output row (blocked fp32 sums)
#pragma unroll
    for (int q = 0; q < BN; ++q) vals[q] = 0.f;
    for (int c = 0; c < nchunks; ++c) {
      const int a = c & 1;
      if (threadIdx.x == 64) WAITP(4, c, &acc_full[a], (c >> 1) & 1);
      else WAITB0(&acc_full[a], (c >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int h = 0; h < BN / 32 && !(P.pad_ & 4); ++h) {  // DG_TMA_DBG bit 2: no drains
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a * BN + h * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 32; ++q) vals[h * 32 + q] += __uint_as_float(r[q]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
    }
    // stage the tile's fp32 sums through shared memory: the last acc_full
    // covers every MMA, so every operand stage has been consumed.  Rows are
    // rotated by 4*row floats against bank conflicts; all warps then write
    // whole rows (coalesced 512 B per row) below
    if (prof_e) g_tprof[5][1][0] = clock64();
    if (kConv) asm volatile("bar.sync 2, 256;" ::: "memory");  // converters done with the stages
    if (!(P.pad_ & 8)) {
      float* part = reinterpret_cast<float*>(smem);  // 128 x 128 fp32 = 64 KiB
      const int lrow = quad * 32 + lane;
#pragma unroll
      for (int q = 0; q < BN; q += 4)
        *reinterpret_cast<float4*>(part + lrow * BN + ((q + 4 * lrow) & (BN - 1))) =
            make_float4(vals[q], vals[q + 1], vals[q + 2], vals[q + 3]);
    }
  }
  if (prof_e) g_tprof[5][2][0] = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();  // every MMA drained and every stage consumed
  if (prof_e) g_tprof[5][3][0] = clock64();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));

  if (P.pad_ & 8) return;  // DG_TMA_DBG bit 3: no epilogue
  const bool has_bias = P.bias.rows != nullptr || P.bias.base != nullptr;
  float* part = reinterpret_cast<float*>(smem);
  cgrp::cluster_group cl = cgrp::this_cluster();
  const bool gs = P.gsplit && S > 1;
  // gsplit: the tile's S CTAs are not co-scheduled as a cluster; each
  // publishes its partial (shared-memory layout verbatim) to the workspace and
  // the last to arrive reduces all S in split order (deterministic)
  const float* gws = gs ? P.ws + (size_t)(blockIdx.x - z) * (BM * BN) : nullptr;
  if (gs) {
    __shared__ int last_sh;
    float4* dst = reinterpret_cast<float4*>(P.ws + (size_t)blockIdx.x * (BM * BN));
    const float4* s4 = reinterpret_cast<const float4*>(part);
    for (int i = threadIdx.x; i < BM * BN / 4; i += blockDim.x) __stcg(dst + i, s4[i]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int t = (int)blockIdx.x / S;
      const int last = atomicAdd(P.cnt + t, 1) == S - 1;
      if (last) P.cnt[t] = 0;  // every split has arrived: leave the counter zero
      last_sh = last;
    }
    __syncthreads();
    if (!last_sh) return;
    __threadfence();
  } else if (S > 1) {
    cl.sync();
  } else {
    __syncthreads();
  }
  if (prof_e) g_tprof[5][4][0] = clock64();
  // cluster: S is a power of two <= 8 and split z reduces rows [z*rows, (z+1)*rows)
  const int rows = gs ? BM : BM / S;
  const int zr = gs ? 0 : z;
  const bool vec = P.c_vec && n0 + BN <= P.N;
  // thread -> fixed 4-column slot ln (NT is a multiple of 32) and rows
  // r0, r0 + RS, ...: a warp writes one whole 512 B row segment per store;
  // U rows per batch with every load issued before the first store.  Kept
  // compact: the kernel's instruction footprint is what the epilogue pays
  constexpr int NT = kConv ? kThreadsConv : kThreads;
  constexpr int RS = NT / 32;
  constexpr int U = 4;
  const int ln = (threadIdx.x & 31) * 4;
  if (!vec) {
    epilogue_scalar(P, part, gws, cl, S, zr, rows, m0, n0, has_bias);
  } else if (gs) {
    // last CTA of a workspace split: whole tile, every split's loads of a row
    // batch in flight before the in-order sum
    constexpr int GU = 2;
    const bool bias_bcast = has_bias && !P.bias.rows && P.bias.ld == 0;
#pragma unroll 1
    for (int rb = (int)(threadIdx.x >> 5); rb < BM; rb += GU * RS) {
      float4 acc4[GU], pv[GU][8];
      float* crow[GU];
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int lm = rb + u * RS;
        const int64_t m = m0 + lm;
        const bool ok = lm < BM && m < P.M;
        crow[u] = ok ? const_cast<float*>(orow(P.C, m)) + n0 + ln : nullptr;
        acc4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok && has_bias)
          acc4[u] = *reinterpret_cast<const float4*>((bias_bcast ? P.bias.base : orow(P.bias, m)) + n0 + ln);
        const int off = lm * BN + ((ln + 4 * lm) & (BN - 1));
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (ok && q < S) pv[u][q] = __ldcg(reinterpret_cast<const float4*>(gws + (size_t)q * (BM * BN) + off));
      }
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        if (!crow[u]) continue;
        float4 v = acc4[u];
        if (P.accumulate) v = f4add(v, *reinterpret_cast<const float4*>(crow[u]));
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < S) v = f4add(v, pv[u][q]);
        if (!(P.pad_ & 2048)) *reinterpret_cast<float4*>(crow[u]) = v;
      }
    }
  } else {
    const bool bias_bcast = has_bias && !P.bias.rows && P.bias.ld == 0;
    const float4 bconst =
        bias_bcast ? *reinterpret_cast<const float4*>(P.bias.base + n0 + ln) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float* src[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) src[q] = q < S && !gs ? (S > 1 ? cl.map_shared_rank(part, q) : part) : part;
#pragma unroll 1
    for (int rb = (int)(threadIdx.x >> 5); rb < rows; rb += U * RS) {
      float4 acc4[U];
      const float* brow[U];
      float* crow[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int lr = rb + u * RS;
        const int64_t m = m0 + zr * rows + lr;
        const bool ok = lr < rows && m < P.M;
        crow[u] = ok ? const_cast<float*>(orow(P.C, m)) + n0 + ln : nullptr;
        brow[u] = ok && has_bias && !bias_bcast ? orow(P.bias, m) + n0 + ln : nullptr;
        acc4[u] = bconst;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!crow[u]) continue;
        if (P.accumulate) acc4[u] = f4add(acc4[u], *reinterpret_cast<const float4*>(crow[u]));
        if (brow[u]) acc4[u] = f4add(acc4[u], *reinterpret_cast<const float4*>(brow[u]));
      }
#pragma unroll 1
      for (int q = 0; q < S; ++q) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int lm = zr * rows + rb + u * RS;
          const int off = lm * BN + ((ln + 4 * lm) & (BN - 1));
          if (rb + u * RS < rows)
            acc4[u] = f4add(acc4[u], gs ? __ldcg(reinterpret_cast<const float4*>(gws + (size_t)q * (BM * BN) + off))
                                        : *reinterpret_cast<const float4*>(src[q] + off));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (crow[u] && !(P.pad_ & 2048)) *reinterpret_cast<float4*>(crow[u]) = acc4[u];
    }
  }
  if (S > 1 && !gs) cl.sync();
  if (prof_e) g_tprof[5][5][0] = clock64();
}

// Persistent form of the lite kernel for single-split problems with many
// tiles (the output-layer logits: ~1.3k tiles, K = 256).  One CTA per SM
// walks tiles blockIdx.x, +gridDim.x, ...; the operand ring runs across tile
// boundaries and the MMA warp alternates two TMEM accumulators, so the
// epilogue warps drain tile i (registers -> staging tile -> coalesced rows)
// while tile i+1 is multiplied.  Same MMA sequence and the same epilogue
// arithmetic as the lite kernel (bit-identical results).
template <bool kAMN, bool kBMN>
__global__ void __launch_bounds__(kThreadsPers, 1) tma_gemm_pers_kernel(const __grid_constant__ TmaGroup G) {
  const TmaProb& PR = G.p[0];
  const CUtensorMap& mAh = PR.mAh;
  const CUtensorMap& mBh = PR.mBh;
  const CUtensorMap& mC = PR.mAl;  // tstore: C's tensor map (the A residual map is unused here)
  const TmaGemmArgs& P = PR.args;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NS = kStagesPers;
  constexpr int SB = 3 * kOpBytes;
  constexpr uint32_t kAcol = 2 * BN;
  __shared__ uint64_t full[NS], empty[NS], conv[NS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (P.M + BM - 1) / BM;
  const int S = P.splits;  // work unit u = (tile u / S, K split u % S); S > 1: workspace partials
  const int ntiles = tiles_m * P.tiles_n * S;  // work units
  const int kt_total = (P.K + BK - 1) / BK;
  __shared__ int last_sh;
  const bool prof = (P.pad_ & 1024) && blockIdx.x == 0;  // DG_TMA_DBG bit 10: CTA 0 wait timeline
#define PWAIT(role, jj, b, ph)                           \
  do {                                                   \
    const long long tb_ = prof ? clock64() : 0;          \
    mbar_wait(b, ph);                                    \
    if (prof && (jj) < 256) {                            \
      g_tprof[role][jj][0] = tb_;                        \
      g_tprof[role][jj][1] = clock64();                  \
    }                                                    \
  } while (0)
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 8);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBh)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_sh)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (P.nowait) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // inputs complete before the preceding grid began
  else pdl_prologue();
  const uint32_t tmem = tmem_sh;
  const uint32_t sbase = su32(smem);
  float* part = reinterpret_cast<float*>(smem + NS * SB);  // output staging tile

  if (warp == 0) {
    if (lane == 0) {
      int j = 0;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
        const int tile = u / S, z = u % S;
        const int m0 = (tile % tiles_m) * BM, n0 = (tile / tiles_m) * BN;
        const int t0 = kt_total * z / S, nkt = kt_total * (z + 1) / S - t0;
        for (int kt = 0; kt < nkt; ++kt, ++j) {
          const int s = j % NS, use = j / NS;
          if (use > 0) PWAIT(0, j, &empty[s], (use - 1) & 1);
          if (P.pad_ & 16) {  // DG_TMA_DBG bit 4: no loads
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_expect_tx(&full[s], 2 * kOpBytes);
          const uint32_t st = sbase + s * SB;
          const int k0 = (t0 + kt) * BK;
          if (!kAMN) {
            tma_2d(st, &mAh, k0, m0, &full[s]);
          } else {
#pragma unroll
            for (int g = 0; g < 4; ++g) tma_2d(st + g * 4096, &mAh, m0 + 32 * g, k0, &full[s]);
          }
          if (!kBMN) {
            tma_2d(st + kOpBytes, &mBh, k0, n0, &full[s]);
          } else {
#pragma unroll
            for (int g = 0; g < 4; ++g) tma_2d(st + kOpBytes + g * 4096, &mBh, n0 + 32 * g, k0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = uidesc(false, kBMN);
      int j = 0, i = 0;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x, ++i) {
        const int z = u % S;
        const int nkt = kt_total * (z + 1) / S - kt_total * z / S;
        const int a = i & 1;
        if (i >= 2) PWAIT(1, i, &acc_empty[a], ((i >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + (uint32_t)(a * BN);
        for (int kt = 0; kt < nkt; ++kt, ++j) {
          const int s = j % NS, use = j / NS;
          PWAIT(2, j, &conv[s], use & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t ah = tmem + kAcol + 64u * (uint32_t)s, al = ah + 32u;
          const uint32_t bh = sbase + s * SB + kOpBytes, bl = bh + kOpBytes;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t ob = kBMN ? ks * 1024 : ks * 32;
            const uint32_t first = (kt == 0 && ks == 0) ? 0u : 1u;
            if (P.pad_ & 1) continue;  // DG_TMA_DBG bit 0: no MMAs
            mma_tf32_ta(acc, ah + 8u * ks, udesc(bh + ob, kBMN), idesc, first);
            mma_tf32_ta(acc, ah + 8u * ks, udesc(bl + ob, kBMN), idesc, 1u);
            mma_tf32_ta(acc, al + 8u * ks, udesc(bh + ob, kBMN), idesc, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[a]);
      }
    }
  } else if (warp >= 10) {
    // B-converter warps 10..13: B's residual into shared memory (elementwise,
    // same swizzled layout)
    const int ct = threadIdx.x - 10 * 32;
    int j = 0;
    for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
      const int nkt = kt_total * (u % S + 1) / S - kt_total * (u % S) / S;
      for (int kt = 0; kt < nkt; ++kt, ++j) {
        const int s = j % NS, use = j / NS;
        mbar_wait(&full[s], use & 1);
        const uint32_t st = sbase + s * SB;
        if (!(P.pad_ & 34)) {  // DG_TMA_DBG bit 1: no conversion (bit 5: no B residual)
#pragma unroll
          for (int i = 0; i < kOpBytes / 16 / 128; ++i) {
            const uint32_t off = (uint32_t)(ct + i * 128) * 16u;
            const float4 x = lds128(st + kOpBytes + off);
            sts128(st + 2 * kOpBytes + off, make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w)));
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else if (warp >= 6) {
    // A-converter warps 6..9 (TMEM lane quadrant warp % 4): A row m split
    // into hi / lo in TMEM lane m
    const int q = warp & 3, m = 32 * q + lane;
    int j = 0;
    for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
      const int nkt = kt_total * (u % S + 1) / S - kt_total * (u % S) / S;
      for (int kt = 0; kt < nkt; ++kt, ++j) {
        const int s = j % NS, use = j / NS;
        if (threadIdx.x == 6 * 32) PWAIT(3, j, &full[s], use & 1);
        else mbar_wait(&full[s], use & 1);
        const uint32_t st = sbase + s * SB;
        if (!(P.pad_ & 514)) {  // bit 9: no A split
          uint32_t hi[32], lo[32];
          if (!kAMN) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float4 x = lds128(st + (uint32_t)m * 128u + ((uint32_t)(c ^ (m & 7)) << 4));
              const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                hi[4 * c + e] = tf32_rn_bits(xv[e]);
                lo[4 * c + e] = __float_as_uint(xv[e] - __uint_as_float(hi[4 * c + e]));
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const float x = lds32(st + (uint32_t)q * 4096u + (uint32_t)k * 128u +
                                    ((uint32_t)(((lane >> 3) ^ (k & 3))) << 5) + ((uint32_t)(lane & 7) << 2));
              hi[k] = tf32_rn_bits(x);
              lo[k] = __float_as_uint(x - __uint_as_float(hi[k]));
            }
          }
          const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + kAcol + 64u * (uint32_t)s;
          tmem_st32(ta, hi);
          tmem_st32(ta + 32u, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else {
    // epilogue warps 2..5 (TMEM lane quadrant warp % 4): 32 columns at a time,
    // registers -> staging buffer (h & 1) -> 8 threads per 128 B row segment
    const int quad = warp & 3, et = threadIdx.x - 64;
    const int lrow = quad * 32 + lane;
    const int c4 = et & 7, r0 = et >> 3;  // store phase: column quad, first row
    const bool has_bias = P.bias.rows != nullptr || P.bias.base != nullptr;
    const bool bias_bcast = has_bias && !P.bias.rows && P.bias.ld == 0;
    int i = 0;
    if (P.tstore) {
      // TMA tensor stores: row lrow's 32 columns of a chunk (+ broadcast bias)
      // into staging buffer h & 1 in the 128 B-swizzled box layout, one
      // thread stores the box; OOB rows / columns are clipped by the TMA unit
      // S > 1: unit u's raw accumulator goes to rows [u*BM, u*BM + BM) of the
      // partial workspace (mC maps it), summed afterwards by split_reduce_kernel
      const uint32_t stg0 = su32(part);
      const bool ext = S > 1;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x, ++i) {
        const int a = i & 1;
        const int tile = u / S;
        const int m0 = (tile % tiles_m) * BM, n0 = (tile / tiles_m) * BN;
        if (threadIdx.x == 64) PWAIT(4, i, &acc_full[a], (i >> 1) & 1);
        else mbar_wait(&acc_full[a], (i >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
        for (int h = 0; h < BN / 32; ++h) {
          uint32_t r[32];
          const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a * BN + h * 32);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(taddr));
          const int nc = n0 + h * 32;
          float bv[32];
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            if (ext) {
              bv[q] = bv[q + 1] = bv[q + 2] = bv[q + 3] = 0.f;
            } else if (has_bias && nc + q + 3 < P.N) {
              const float4 t = *reinterpret_cast<const float4*>(P.bias.base + nc + q);
              bv[q] = t.x, bv[q + 1] = t.y, bv[q + 2] = t.z, bv[q + 3] = t.w;
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) bv[q + e] = has_bias && nc + q + e < P.N ? P.bias.base[nc + q + e] : 0.f;
            }
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (h == BN / 32 - 1) {
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[a]);
          }
          // buffer h & 1 was last read by the store of chunk h - 2
          if (threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const uint32_t stg = stg0 + (uint32_t)((h & 1) * BM * 32 * 4);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            sts128(stg + (uint32_t)lrow * 128u + ((uint32_t)(c ^ (lrow & 7)) << 4),
                   make_float4(bv[4 * c] + __uint_as_float(r[4 * c]), bv[4 * c + 1] + __uint_as_float(r[4 * c + 1]),
                               bv[4 * c + 2] + __uint_as_float(r[4 * c + 2]),
                               bv[4 * c + 3] + __uint_as_float(r[4 * c + 3])));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (threadIdx.x == 64 && !(P.pad_ & 8)) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&mC)),
                "r"(ext ? h * 32 : nc), "r"(ext ? u * BM : m0), "r"(stg)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (prof && threadIdx.x == 64 && i < 256) g_tprof[5][i][0] = clock64();
      }
      if (threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    if (S > 1 && !P.tstore) {
      // split units: the raw accumulator goes to workspace slot u (row-major
      // 128 x 128); the tile's last unit to arrive adds bias, C and the S
      // partials in split order (the cluster kernels' arithmetic and order)
      const int ew = warp - 2;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x, ++i) {
        const int a = i & 1;
        const int tile = u / S;
        const int m0 = (tile % tiles_m) * BM, n0 = (tile / tiles_m) * BN;
        if (threadIdx.x == 64) PWAIT(4, i, &acc_full[a], (i >> 1) & 1);
        else mbar_wait(&acc_full[a], (i >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        float* slot = P.ws + (size_t)u * (BM * BN) + (size_t)lrow * BN;
#pragma unroll 1
        for (int h = 0; h < BN / 32; ++h) {
          uint32_t r[32];
          const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a * BN + h * 32);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (h == BN / 32 - 1) {
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[a]);
          }
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            __stcg(reinterpret_cast<float4*>(slot + h * 32 + q),
                   make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]), __uint_as_float(r[q + 2]),
                               __uint_as_float(r[q + 3])));
        }
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          const int last = atomicAdd(P.cnt + tile, 1) == S - 1;
          if (last) P.cnt[tile] = 0;  // every split has arrived: leave the counter zero
          last_sh = last;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (last_sh) {
          __threadfence();
          const float* base = P.ws + (size_t)tile * S * (BM * BN);
          const int ln = lane * 4;
          const bool vec = P.c_vec && n0 + BN <= P.N;
          const float4 bconst = vec && bias_bcast ? *reinterpret_cast<const float4*>(P.bias.base + n0 + ln)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
          for (int lr0 = ew; lr0 < BM; lr0 += 8) {
            // rows lr0 and lr0 + 4: the partials in batches of 8 (all loads of
            // a batch in flight), summed in split order
            float4 acc[2];
            bool ok[2];
            float* crow[2];
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              const int64_t m = m0 + lr0 + 4 * w;
              ok[w] = m < P.M;
              crow[w] = ok[w] ? const_cast<float*>(orow(P.C, m)) : nullptr;
              acc[w] = bconst;
              if (ok[w] && vec) {
                if (P.accumulate) acc[w] = f4add(acc[w], *reinterpret_cast<const float4*>(crow[w] + n0 + ln));
                if (has_bias && !bias_bcast)
                  acc[w] = f4add(acc[w], *reinterpret_cast<const float4*>(orow(P.bias, m) + n0 + ln));
              }
            }
            float4 ps[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};  // scalar path
#pragma unroll 1
            for (int qb = 0; qb < S; qb += 8) {
              float4 pv[2][8];
#pragma unroll
              for (int w = 0; w < 2; ++w)
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  if (qb + q < S)
                    pv[w][q] = __ldcg(reinterpret_cast<const float4*>(base + (size_t)(qb + q) * (BM * BN) +
                                                                      (lr0 + 4 * w) * BN + ln));
#pragma unroll
              for (int w = 0; w < 2; ++w)
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  if (qb + q < S) {
                    if (vec) acc[w] = f4add(acc[w], pv[w][q]);
                    else ps[w] = f4add(ps[w], pv[w][q]);
                  }
            }
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              if (!ok[w]) continue;
              if (vec) {
                *reinterpret_cast<float4*>(crow[w] + n0 + ln) = acc[w];
              } else {
                const int64_t m = m0 + lr0 + 4 * w;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int64_t n = n0 + ln + e;
                  if (n >= P.N) continue;
                  float v = reinterpret_cast<const float*>(&ps[w])[e];
                  if (has_bias) v += orow(P.bias, m)[n];
                  if (P.accumulate) v += crow[w][n];
                  crow[w][n] = v;
                }
              }
            }
          }
        }
        if (prof && threadIdx.x == 64 && i < 256) g_tprof[5][i][0] = clock64();
      }
    }
    for (int tile = P.tstore || S > 1 ? ntiles : blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
      const int a = i & 1;
      const int m0 = (tile % tiles_m) * BM, n0 = (tile / tiles_m) * BN;
      const bool vec = P.c_vec && n0 + BN <= P.N;
      float4 bpre[BN / 32];  // broadcast bias of this thread's column quad in each chunk, loaded ahead
#pragma unroll
      for (int h = 0; h < BN / 32; ++h)
        bpre[h] = vec && bias_bcast ? *reinterpret_cast<const float4*>(P.bias.base + n0 + h * 32 + 4 * c4)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      if (threadIdx.x == 64) PWAIT(4, i, &acc_full[a], (i >> 1) & 1);
      else mbar_wait(&acc_full[a], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int h = 0; h < BN / 32; ++h) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a * BN + h * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const bool pe = prof && threadIdx.x == 64 && i >= 1 && i <= 3;
        if (pe) g_tprof[4][64 + i * 16 + h * 4 + 0][0] = clock64();
        if (h == BN / 32 - 1) {  // accumulator drained: the MMA warp may refill it
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[a]);
        }
        float* stg = part + (h & 1) * (BM * 32);
#pragma unroll
        for (int q = 0; q < 32; q += 4)
          *reinterpret_cast<float4*>(stg + lrow * 32 + ((q + 4 * lrow) & 31)) =
              make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]), __uint_as_float(r[q + 2]),
                          __uint_as_float(r[q + 3]));
        // buffer h & 1 complete; its previous contents (chunk h - 2) were
        // stored before every thread passed the barrier of chunk h - 1
        if (pe) g_tprof[4][64 + i * 16 + h * 4 + 1][0] = clock64();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (pe) g_tprof[4][64 + i * 16 + h * 4 + 2][0] = clock64();
        const int nc = n0 + h * 32;
        if (P.pad_ & 8) continue;  // DG_TMA_DBG bit 3: no global stores
        if (vec) {
          const float4 bconst = bpre[h];
#pragma unroll 4
          for (int lr = r0; lr < BM; lr += 16) {
            const int64_t m = m0 + lr;
            if (m >= P.M) break;
            float* crow = const_cast<float*>(orow(P.C, m)) + nc + 4 * c4;
            float4 v = bconst;
            if (P.accumulate) v = f4add(v, *reinterpret_cast<const float4*>(crow));
            if (has_bias && !bias_bcast) v = f4add(v, *reinterpret_cast<const float4*>(orow(P.bias, m) + nc + 4 * c4));
            v = f4add(v, *reinterpret_cast<const float4*>(stg + lr * 32 + ((4 * c4 + 4 * lr) & 31)));
            *reinterpret_cast<float4*>(crow) = v;
          }
          if (pe) g_tprof[4][64 + i * 16 + h * 4 + 3][0] = clock64();
        } else {
          for (int e = et; e < BM * 32; e += 128) {
            const int lr = e >> 5, c = e & 31;
            const int64_t m = m0 + lr, n = nc + c;
            if (m >= P.M || n >= P.N) continue;
            float v = 0.f;
            v += stg[lr * 32 + (((c & ~3) + 4 * lr) & 31) + (c & 3)];
            float* crow = const_cast<float*>(orow(P.C, m));
            if (has_bias) v += orow(P.bias, m)[n];
            if (P.accumulate) v += crow[n];
            crow[n] = v;
          }
        }
      }
      if (prof && threadIdx.x == 64 && i < 256) g_tprof[5][i][0] = clock64();
    }
  }
#undef PWAIT
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Sum of the persistent kernel's split partials (workspace rows u*BM.. of
// unit u = tile*S + z, row-major BM x BN) into C, in split order, with the
// cluster kernels' arithmetic: bias + C + row bias + p_0 + ... + p_{S-1}
// (vector path) / p_0 + ... + bias + C (scalar path)
__global__ void split_reduce_kernel(const __grid_constant__ TmaGemmArgs P) {
  pdl_prologue();
  const int S = P.splits, tiles_m = (P.M + BM - 1) / BM;
  const int nq = (P.N + 3) >> 2;
  const int64_t total = (int64_t)P.M * nq;
  const bool has_bias = P.bias.rows != nullptr || P.bias.base != nullptr;
  const bool bias_bcast = has_bias && !P.bias.rows && P.bias.ld == 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(t / nq), n = 4 * (int)(t - (int64_t)m * nq);
    const int tile = m / BM + (n / BN) * tiles_m;
    const float* p0 = P.ws + ((size_t)tile * S * BM + (m % BM)) * BN + (n % BN);
    float* crow = const_cast<float*>(orow(P.C, m));
    if (P.c_vec && n + 3 < P.N) {
      float4 v = bias_bcast ? *reinterpret_cast<const float4*>(P.bias.base + n) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (P.accumulate) v = f4add(v, *reinterpret_cast<const float4*>(crow + n));
      if (has_bias && !bias_bcast) v = f4add(v, *reinterpret_cast<const float4*>(orow(P.bias, m) + n));
      for (int q = 0; q < S; ++q) v = f4add(v, __ldcg(reinterpret_cast<const float4*>(p0 + (size_t)q * BM * BN)));
      *reinterpret_cast<float4*>(crow + n) = v;
    } else {
      for (int e = 0; e < 4 && n + e < P.N; ++e) {
        float v = 0.f;
        for (int q = 0; q < S; ++q) v += __ldcg(p0 + (size_t)q * BM * BN + e);
        if (has_bias) v += orow(P.bias, m)[n + e];
        if (P.accumulate) v += crow[n + e];
        crow[n + e] = v;
      }
    }
  }
}

// lo[r][c] = x - tf32(x) for up to two rows x cols blocks (A and B of one
// GEMM in a single launch), row stride ld; dst dense with stride cols_p
struct SplitJob {
  const float* src;
  float* dst;
  int64_t ld, rows, cols, cols_p;
};
__global__ void split_lo_kernel(SplitJob j0, SplitJob j1, int n_jobs) {
  pdl_prologue();
  const int64_t t0 = j0.rows * (j0.cols_p >> 2);
  const int64_t total = t0 + (n_jobs > 1 ? j1.rows * (j1.cols_p >> 2) : 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const bool second = i >= t0;
    const SplitJob& j = second ? j1 : j0;
    const int64_t q = second ? i - t0 : i;
    const int64_t c4 = j.cols_p >> 2;
    const int64_t r = q / c4, c = (q - r * c4) * 4;
    const float* s = j.src + r * j.ld + c;
    float4 o;
    float* op = reinterpret_cast<float*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float x = c + k < j.cols ? s[k] : 0.f;
      op[k] = tf32_rn_lo_of_raw(x);
    }
    *reinterpret_cast<float4*>(j.dst + r * j.cols_p + c) = o;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// rows x cols fp32 block, row stride ld floats; box {32, box_rows} (K-major:
// 32 k x 128 rows, SWIZZLE_128B) or {32, 32} (MN-major, SWIZZLE_128B_ATOM_32B)
struct MapKey {
  const float* base;
  int64_t ld, rows, cols;
  bool mn;
  bool operator==(const MapKey& o) const {
    return base == o.base && ld == o.ld && rows == o.rows && cols == o.cols && mn == o.mn;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = reinterpret_cast<uintptr_t>(k.base) * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)k.ld + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
    h ^= (uint64_t)k.rows * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
    h ^= (uint64_t)k.cols * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
    return (size_t)(h ^ (k.mn ? 0x27D4EB2F165667C5ull : 0));
  }
};

bool make_map_uncached(CUtensorMap* m, const float* base, int64_t ld, int64_t rows, int64_t cols, bool mn);

// Tensor maps are pure functions of (base, ld, rows, cols, layout); the
// arenas are reused step after step, so the same blocks recur and the
// driver-side encode (several us each) is done once per distinct block
bool make_map(CUtensorMap* m, const float* base, int64_t ld, int64_t rows, int64_t cols, bool mn) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{base, ld, rows, cols, mn};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *m = it->second;
      return true;
    }
  }
  if (!make_map_uncached(m, base, ld, rows, cols, mn)) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}

bool make_map_uncached(CUtensorMap* m, const float* base, int64_t ld, int64_t rows, int64_t cols, bool mn) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, mn ? 32u : 128u};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int tma_prof_read(long long* out) {
  return cudaMemcpyFromSymbol(out, g_tprof, sizeof(g_tprof)) == cudaSuccess ? 0 : -1;  // [6][256][2]
}

bool tma_lite_enabled();

// whole-split accumulation in TMEM (no blocked drains) for short splits: the
// error stays at a few 1e-6 relative, the size of the fp32 reference's own
// summation error (tools/tma_bench.cu; long splits keep the blocked drains)
static bool lite_ok(bool a_tmem, int K, int S) {
  const int kt = (K + BK - 1) / BK;
  const int per = ((kt + S - 1) / S) * BK;
  return a_tmem && S <= 4 && per <= (S == 1 ? kLiteMaxK : kLiteMaxKSplit) && tma_lite_enabled();
}

bool tma_lite_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TMA_LITE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tma_at_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TMA_AT");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tma_conv_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TMA_CONV");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tma_gemm_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TMA");
    return !(e && e[0] == '0');
  }();
  return on && tc_gemm_enabled();
}

bool tma_pers_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TMA_PERS");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int sm_count() {
  static const int n = [] {
    int d = 0, v = 0;
    if (cudaGetDevice(&d) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess)
      v = 148;
    return v > 0 ? v : 148;
  }();
  return n;
}

constexpr int kPersMaxSplit = 16;
// work units per SM below which the persistent kernel is not used
// (DG_TMA_PERS_MIN, default 4)
static int pers_min_units() {
  static const int v = [] {
    const char* e = getenv("DG_TMA_PERS_MIN");
    return e ? atoi(e) : 4;
  }();
  return v;
}

bool tma_tstore_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TMA_TSTORE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tma_gsplit_enabled() {
  static const bool on = [] {
    const char* e = getenv("DG_TMA_GSPLIT");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int tma_kernel_index(const TmaGemmPlan& p);
using TmaKernel = void (*)(const TmaGroup);
static TmaKernel tma_kernel(int ki);
static int tma_smem(bool lite, bool a_tmem, bool conv, bool pers = false) {
  return pers ? kSmemPers : lite ? kSmemLite : a_tmem ? kSmemAT : conv ? kSmemConv : kSmem;
}
static bool tma_attr(int ki, int smem) {
  static bool attr[20] = {};
  if (!attr[ki]) {
    if (cudaFuncSetAttribute(tma_kernel(ki), cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return false;
    attr[ki] = true;
  }
  return true;
}

// clusters of S CTAs of kernel variant ki that can be resident at once
static int max_clusters(int ki, int S, int smem, int threads) {
  static std::mutex mu;
  static int cache[20][9] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (cache[ki][S]) return cache[ki][S];
  int n = 0;
  if (tma_attr(ki, smem)) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(S * 256);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, tma_kernel(ki), &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
  }
  cache[ki][S] = n > 0 ? n : 1;
  return cache[ki][S];
}

// Workspace split-K instead of clusters when the S-CTA clusters of a launch
// would not all be co-resident (cluster placement is per GPC: on 148 SMs only
// ~32 four-CTA clusters of a one-CTA-per-SM kernel fit, so 34 clusters run in
// two rounds) while the same CTAs without clusters fit in one round.
static bool use_gsplit(int tiles, int S, bool a_tmem, int K, int64_t ws_floats, int cnt_cap) {
  if (S < 2 || !tma_gsplit_enabled() || cnt_cap < tiles || (int64_t)tiles * S * (BM * BN) > ws_floats) return false;
  const bool lite = lite_ok(a_tmem, K, S);
  const bool conv = tma_conv_enabled();
  const int c = lite ? 2 : 1;
  if (tiles * S > 148 * c) return false;
  TmaGemmPlan q{};
  q.lite = lite;
  q.a_tmem = a_tmem;
  q.conv = conv;
  const int ki = tma_kernel_index(q);
  const int mc = max_clusters(ki, S, tma_smem(lite, a_tmem, conv), conv ? kThreadsConv : kThreads);
  return tiles > mc;
}

int64_t tma_lo_floats(int64_t rows, int64_t cols) { return rows * ((cols + 3) & ~int64_t(3)); }

bool tma_gemm_make(const TmaOperands& o, TmaGemmPlan* out) {
  TmaGemmPlan p{};
  p.a_mn = o.a_mn;
  p.b_mn = o.b_mn;
  TmaGemmArgs& a = p.args;
  a.M = o.M;
  a.N = o.N;
  a.K = o.K;
  a.C = o.C;
  a.bias = o.bias;
  a.accumulate = o.accumulate;
  // 16 B epilogue accesses: a dense C aligned with ld % 4 == 0, or a row table
  // whose rows are arena / parameter slots (64 B aligned, rows of N floats
  // apart) with N % 4 == 0
  a.c_vec = (o.C.rows ? o.N % 4 == 0
                      : (reinterpret_cast<uintptr_t>(o.C.base) % 16 == 0) && o.C.ld % 4 == 0) &&
            (!o.bias.base || o.bias.rows || (reinterpret_cast<uintptr_t>(o.bias.base) % 16 == 0 && o.bias.ld % 4 == 0));
  // operand blocks: A is (M rows x K) or (K rows x M); B is (N x K) or (K x N)
  const int64_t ar = o.a_mn ? o.K : o.M, ac = o.a_mn ? o.M : o.K;
  const int64_t br = o.b_mn ? o.K : o.N, bc = o.b_mn ? o.N : o.K;
  const int64_t acp = (ac + 3) & ~int64_t(3), bcp = (bc + 3) & ~int64_t(3);
  p.a_src = o.A;
  p.a_ld = o.lda;
  p.a_rows = ar;
  p.a_cols = ac;
  p.a_colsp = acp;
  p.a_lo = o.A_lo;
  p.b_src = o.B;
  p.b_ld = o.ldb;
  p.b_rows = br;
  p.b_cols = bc;
  p.b_colsp = bcp;
  p.b_lo = o.B_lo;
  p.conv = tma_conv_enabled();
  p.a_tmem = p.conv && tma_at_enabled();
  if (!make_map(&p.mAh, o.A, o.lda, ar, ac, o.a_mn) || !make_map(&p.mBh, o.B, o.ldb, br, bc, o.b_mn)) return false;
  if (p.conv) {  // residuals formed in shared memory: no lo copies, no lo maps
    p.mAl = p.mAh;
    p.mBl = p.mBh;
  } else if (!make_map(&p.mAl, o.A_lo, acp, ar, ac, o.a_mn) || !make_map(&p.mBl, o.B_lo, bcp, br, bc, o.b_mn)) {
    return false;
  }
  a.tiles_n = (o.N + BN - 1) / BN;
  const int tiles = ((o.M + BM - 1) / BM) * a.tiles_n;
  const int kt = (o.K + BK - 1) / BK;
  p.ws_floats = o.ws ? o.ws_floats : 0;
  p.cnt_cap = o.cnt ? o.cnt_cap : 0;
  a.ws = o.ws;
  a.cnt = o.cnt;
  // split-K (a cluster of S CTAs per tile) for the best wave efficiency on
  // 148 SMs (one CTA per SM); each split keeps >= 4 k-tiles
  // cost model: waves x (fixed per-CTA cost ~ 4 k-tiles + k-tiles per split)
  int S = 1;
  double best = 1e30;
  for (int s2 = 1; s2 <= 8; s2 *= 2) {
    if (s2 > 1 && kt < 4 * s2) break;
    const int units = tiles * s2;
    const double cost = (double)((units + 147) / 148) * (4.0 + (double)kt / s2);
    if (cost < best * 0.97) {
      best = cost;
      S = s2;
    }
  }
  a.gsplit = use_gsplit(tiles, S, p.a_tmem, o.K, p.ws_floats, p.cnt_cap) ? 1 : 0;
  // DG_TMA_DBG (diagnostics, tools/tma_bench): bits 0-4 skip MMAs /
  // conversion / drains / epilogue / loads, bit 6 plain arrives for commits,
  // bit 7 no proxy fence, bit 10 CTA-0 wait timeline, bits 11-12 skip
  // epilogue stores / reductions, bits 16-19 force the split factor
  static const int dbg = [] {
    const char* e = getenv("DG_TMA_DBG");
    return e ? (int)strtol(e, nullptr, 0) : 0;
  }();
  a.pad_ = dbg & 0xFFFF;
  if ((dbg >> 16) & 0xF) S = (dbg >> 16) & 0xF;
  if ((dbg >> 20) & 2) a.gsplit = p.ws_floats >= (int64_t)tiles * S * (BM * BN) && p.cnt_cap >= tiles;  // bit 21
  if (a.gsplit && (int64_t)tiles * S * (BM * BN) > p.ws_floats) S = 1;
  if (!a.gsplit && (S & (S - 1))) S = 1;  // cluster splits reduce BM / S rows each
  if (S == 1) a.gsplit = 0;
  a.splits = S;
  p.ctas = tiles * S;
  p.lite = lite_ok(p.a_tmem, o.K, S);
  // persistent CTAs once the lite-sized work units (tile x K split) fill more
  // than ~two rounds of two CTAs per SM: the split factor minimises rounds x
  // (k-tiles per unit + a partial-tile cost per split)
  p.pers = false;
  if (tma_pers_enabled() && p.a_tmem && !(dbg & 0xF0000)) {
    const int sm = sm_count();
    double best_c = 1e30;
    int best_s = 0;
    // DG_TMA_PERS_SPLIT=0: persistent kernel for unsplit problems only
    static const bool split_on = [] {
      const char* e = getenv("DG_TMA_PERS_SPLIT");
      return !(e && e[0] == '0');
    }();
    for (int s2 = 1; s2 <= (split_on ? kPersMaxSplit : 1); ++s2) {
      const int per = (kt + s2 - 1) / s2;
      if (per * BK > (s2 == 1 ? kLiteMaxK : kLiteMaxKSplit) || !tma_lite_enabled()) continue;
      if (s2 > 1 && (kt < 4 * s2 || !tma_gsplit_enabled() || p.cnt_cap < tiles ||
                     (int64_t)tiles * s2 * (BM * BN) > p.ws_floats))
        continue;
      const int units = tiles * s2;
      if (units <= pers_min_units() * sm) continue;
      const double c = (double)((units + sm - 1) / sm) * (per + (s2 > 1 ? 0.25 * s2 : 0.0));
      if (c < best_c) {
        best_c = c;
        best_s = s2;
      }
    }
    if (best_s) {
      p.pers = true;
      p.lite = true;
      S = best_s;
      a.splits = S;
      a.gsplit = S > 1;
      p.ctas = tiles * S;
    }
  }
  a.tstore = 0;
  // split units: partial tiles through TMA stores into the workspace (a
  // tensor map over units*BM rows of BN floats), reduced by a second launch
  if (p.pers && S > 1 && tma_tstore_enabled() &&
      make_map(&p.mAl, o.ws, BN, (int64_t)p.ctas * BM, BN, false))
    a.tstore = 1;
  const bool bias_ok = !(o.bias.base || o.bias.rows) || (o.bias.base && !o.bias.rows && o.bias.ld == 0 &&
                                                          reinterpret_cast<uintptr_t>(o.bias.base) % 16 == 0);
  if (p.pers && S == 1 && tma_tstore_enabled() && !o.accumulate && !o.C.rows && o.C.base && bias_ok &&
      reinterpret_cast<uintptr_t>(o.C.base) % 16 == 0 && o.C.ld % 4 == 0 &&
      make_map(&p.mAl, o.C.base, o.C.ld, o.M, o.N, false))
    a.tstore = 1;
  if (dbg & 0x100000)  // DG_TMA_DBG bit 20: log each planned GEMM
    fprintf(stderr, "[tma] M %d N %d K %d a_mn %d b_mn %d acc %d bias %d rows %d split %d ctas %d\n", o.M, o.N, o.K,
            (int)o.a_mn, (int)o.b_mn, o.accumulate, (int)(o.bias.base || o.bias.rows), (int)(o.C.rows != nullptr), S,
            p.ctas);
  p.flops = 2.0 * o.M * (double)o.N * o.K;
  *out = p;
  return true;
}

static int tma_kernel_index(const TmaGemmPlan& p) {  // (declared above)
  return (p.pers ? 16 : p.lite ? 12 : p.a_tmem ? 8 : p.conv ? 4 : 0) + (p.a_mn ? 2 : 0) + (p.b_mn ? 1 : 0);
}

static TmaKernel tma_kernel(int ki) {
  static const TmaKernel table[20] = {
      tma_gemm_kernel<false, false, false>,      tma_gemm_kernel<false, true, false>,
      tma_gemm_kernel<true, false, false>,       tma_gemm_kernel<true, true, false>,
      tma_gemm_kernel<false, false, true>,       tma_gemm_kernel<false, true, true>,
      tma_gemm_kernel<true, false, true>,        tma_gemm_kernel<true, true, true>,
      tma_gemm_kernel<false, false, true, true>, tma_gemm_kernel<false, true, true, true>,
      tma_gemm_kernel<true, false, true, true>,  tma_gemm_kernel<true, true, true, true>,
      tma_gemm_kernel<false, false, true, true, true>, tma_gemm_kernel<false, true, true, true, true>,
      tma_gemm_kernel<true, false, true, true, true>,  tma_gemm_kernel<true, true, true, true, true>,
      tma_gemm_pers_kernel<false, false>,              tma_gemm_pers_kernel<false, true>,
      tma_gemm_pers_kernel<true, false>,               tma_gemm_pers_kernel<true, true>};
  return table[ki];
}

static int tma_launch(const TmaGemmPlan* const* ps, int n, cudaStream_t s) {
  const TmaGemmPlan& p = *ps[0];
  const int ki = tma_kernel_index(p);
  const TmaKernel k = tma_kernel(ki);
  const int smem = tma_smem(p.lite, p.a_tmem, p.conv, p.pers);
  if (!tma_attr(ki, smem)) return -1;
  static TmaGroup G;  // launch arguments are copied at launch
  G.n = n;
  int ctas = 0;
  for (int i = 0; i < n; ++i) {
    G.p[i].mAh = ps[i]->mAh;
    G.p[i].mAl = ps[i]->mAl;
    G.p[i].mBh = ps[i]->mBh;
    G.p[i].mBl = ps[i]->mBl;
    G.p[i].args = ps[i]->args;
    G.p[i].cta0 = ctas;
    ctas += ps[i]->ctas;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.pers ? std::min(ctas, p.grid_cap > 0 ? std::min(p.grid_cap, sm_count()) : sm_count()) : ctas);
  cfg.blockDim = dim3(p.pers ? kThreadsPers : p.conv ? kThreadsConv : kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.args.gsplit ? 1 : p.args.splits;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, G) == cudaSuccess ? 1 : -1;
}

int launch_tma_gemm(const TmaGemmPlan& p, bool split_a, bool split_b, cudaStream_t s) {
  int n = 0;
  if (p.conv) split_a = split_b = false;
  {
    SplitJob jobs[2];
    int nj = 0;
    if (split_a) jobs[nj++] = SplitJob{p.a_src, p.a_lo, p.a_ld, p.a_rows, p.a_cols, p.a_colsp};
    if (split_b) jobs[nj++] = SplitJob{p.b_src, p.b_lo, p.b_ld, p.b_rows, p.b_cols, p.b_colsp};
    if (nj) {
      int64_t tot = 0;
      for (int q = 0; q < nj; ++q) tot += jobs[q].rows * (jobs[q].cols_p / 4);
      launch_k(split_lo_kernel, (int)std::min<int64_t>((tot + 255) / 256, 148 * 8), 256, 0, s, jobs[0], jobs[nj - 1], nj);
      ++n;
    }
  }
  const TmaGemmPlan* one = &p;
  const int r = tma_launch(&one, 1, s);
  if (r < 0) return -1;
  if (p.pers && p.args.splits > 1 && p.args.tstore) {
    const int64_t total = (int64_t)p.args.M * ((p.args.N + 3) / 4);
    launch_k(split_reduce_kernel, (int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, s, p.args);
    ++n;
  }
  return n + r;
}

bool tma_gemm_groupable(const TmaGemmPlan& a, const TmaGemmPlan& b) {
  if (a.pers || b.pers) return false;
  if (!a.conv || !b.conv || a.a_tmem != b.a_tmem || a.a_mn != b.a_mn || a.b_mn != b.b_mn) return false;
  if (a.args.C.rows || b.args.C.rows) return false;
  // output blocks must not overlap (problems of a group run concurrently)
  auto lo = [](const TmaGemmPlan& p) { return p.args.C.base; };
  auto hi = [](const TmaGemmPlan& p) { return p.args.C.base + (int64_t)(p.args.M - 1) * p.args.C.ld + p.args.N; };
  return hi(a) <= lo(b) || hi(b) <= lo(a);
}

void tma_gemm_regroup(TmaGemmPlan* const* ps, int n) {
  // one split factor for the group: waves x (fixed ~4 k-tiles + longest split)
  int tiles = 0, kt_max = 0, kt_min = 1 << 30;
  for (int i = 0; i < n; ++i) {
    const TmaGemmArgs& a = ps[i]->args;
    tiles += ((a.M + BM - 1) / BM) * a.tiles_n;
    const int kt = (a.K + BK - 1) / BK;
    kt_max = std::max(kt_max, kt);
    kt_min = std::min(kt_min, kt);
  }
  int S = 1;
  double best = 1e30;
  for (int s2 = 1; s2 <= 8; s2 *= 2) {
    if (s2 > 1 && kt_min < 4 * s2) break;
    const double cost = (double)((tiles * s2 + 147) / 148) * (4.0 + (double)kt_max / s2);
    if (cost < best * 0.97) {
      best = cost;
      S = s2;
    }
  }
  // workspace split-K when every problem shares one workspace
  bool gs = true;
  int K_max = 0;
  for (int i = 0; i < n; ++i) {
    gs = gs && ps[i]->args.ws == ps[0]->args.ws && ps[i]->args.cnt == ps[0]->args.cnt;
    K_max = std::max(K_max, ps[i]->args.K);
  }
  gs = gs && use_gsplit(tiles, S, ps[0]->a_tmem, K_max, ps[0]->ws_floats, ps[0]->cnt_cap);
  for (int i = 0; i < n; ++i) {
    TmaGemmArgs& a = ps[i]->args;
    a.gsplit = gs ? 1 : 0;
    a.splits = S;
    ps[i]->ctas = ((a.M + BM - 1) / BM) * a.tiles_n * S;
    ps[i]->lite = lite_ok(ps[i]->a_tmem, a.K, S);
    ps[i]->pers = false;
  }
}

int launch_tma_gemm_group(const TmaGemmPlan* const* ps, int n, cudaStream_t s) {
  if (n <= 0) return 0;
  if (n > kTmaGroup) return -1;
  return tma_launch(ps, n, s);
}

}  // namespace dg
