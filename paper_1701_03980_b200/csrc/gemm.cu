// Grouped FP32 SIMT GEMM over gathered rows for the batched affine
// contractions (ops.py:323-357: out = b + sum_k x_k W_k^T; dW += G^T x;
// dx += G W).
//
//   for each problem p:  C_p[M x N] (= | +=) sum_seg A_seg(m,k) B_seg(k,n) (+ bias_m(n))
//
// One launch covers a list of independent problems (both layers' affines of
// a recurrence level, every dX term of a level, ...).  Operands are addressed
// row by row (device row-pointer table or base+ld), so a problem spans every
// node of a batched group, batch-1 broadcast operands (rows repeating one
// pointer) and every use of a parameter across the graph (weight-gradient
// aggregation).  K is a concatenation of up to 4 segments (multi-term affine).
//
// Split-K is deterministic without a second launch: each split CTA writes its
// partial tile to the workspace, bumps a per-tile counter, and the CTA that
// arrives last reduces the partials in split order and runs the epilogue.
// fp32 throughout for the rtol 1e-4 parity bar.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace cgrp = cooperative_groups;

namespace dg {
namespace {

__device__ __forceinline__ const float* op_row(const Operand& o, int64_t i) {
  return o.rows ? o.rows[i] : o.base + i * o.ld;
}

template <int BM, int BN, int BK, int TM, int TN>
struct Cfg {
  static constexpr int kThreads = (BM / TM) * (BN / TN);
  static constexpr int kApad = BM + 4;
  static constexpr int kBpad = BN + 4;
  static_assert((BM * BK) % (4 * kThreads) == 0 && (BK * BN) % (4 * kThreads) == 0, "tile/threads");
};

// Tile loader: ROWS x COLS tile in source order (source row r holds COLS
// contiguous elements).  Vector (float4) or scalar path chosen at run time.
template <int ROWS, int COLS, int THREADS>
struct TileLoad {
  static constexpr int kPer = (ROWS * COLS) / THREADS;
  float v[kPer];

  // cache: optional shared-memory copy of the tile's ROWS row pointers
  __device__ __forceinline__ void load(const Operand& op, bool vec, int64_t row0, int64_t row_lim, int64_t col0,
                                       int64_t col_lim, const float* const* cache = nullptr) {
    const int tid = threadIdx.x;
    auto row = [&](int r, int64_t gr) { return cache ? cache[r] : op_row(op, gr); };
    if (vec) {
#pragma unroll
      for (int i = 0; i < kPer / 4; ++i) {
        const int idx = (tid + i * THREADS) * 4;
        const int r = idx / COLS, c = idx % COLS;
        const int64_t gr = row0 + r, gc = col0 + c;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gr < row_lim && gc < col_lim) x = __ldg(reinterpret_cast<const float4*>(row(r, gr) + gc));
        v[i * 4 + 0] = x.x;
        v[i * 4 + 1] = x.y;
        v[i * 4 + 2] = x.z;
        v[i * 4 + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kPer / 4; ++i) {
        const int idx = (tid + i * THREADS) * 4;
        const int r = idx / COLS, c = idx % COLS;
        const int64_t gr = row0 + r;
        const float* rp = gr < row_lim ? row(r, gr) : nullptr;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t gc = col0 + c + q;
          v[i * 4 + q] = (rp && gc < col_lim) ? __ldg(rp + gc) : 0.f;
        }
      }
    }
  }

  // store into smem tile S[k][mn] (pitch P); kTrans: source rows are the mn axis
  template <bool kTrans, int P>
  __device__ __forceinline__ void store(float* S) const {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < kPer / 4; ++i) {
      const int idx = (tid + i * THREADS) * 4;
      const int r = idx / COLS, c = idx % COLS;
      if (kTrans) {
#pragma unroll
        for (int q = 0; q < 4; ++q) S[(c + q) * P + r] = v[i * 4 + q];
      } else {
        *reinterpret_cast<float4*>(S + r * P + c) = make_float4(v[i * 4], v[i * 4 + 1], v[i * 4 + 2], v[i * 4 + 3]);
      }
    }
  }
};

// kCl: split-K across the CTAs of a thread-block cluster (cluster size =
// splits, one cluster per output tile); partial tiles are reduced through
// distributed shared memory in fixed split order.  Otherwise split-K goes
// through global partials + a per-tile arrival counter (last CTA reduces).
template <int BM, int BN, int BK, int TM, int TN, bool kAK, bool kBN, bool kCl>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, TM, TN>::kThreads)
    gemm_group_kernel(const GemmProblem* __restrict__ probs, int n_probs, float* __restrict__ work,
                      int* __restrict__ counters) {
  pdl_prologue();
  using C = Cfg<BM, BN, BK, TM, TN>;
  __shared__ __align__(16) float As[2][BK * C::kApad];
  __shared__ __align__(16) float Bs[2][BK * C::kBpad];
  __shared__ __align__(16) float red[kCl ? BM * BN : 4];
  __shared__ GemmProblem P;
  __shared__ int s_last;
  // per-segment row pointers of the tile's fixed rows (A rows when A is
  // m-major, B rows when B is n-major): one global load per element later
  __shared__ const float* rowA[4][kAK ? 1 : BM];
  __shared__ const float* rowB[4][kBN ? BN : 1];

  // locate this CTA's problem (problems are few; linear scan of cta0)
  int p = 0;
  while (p + 1 < n_probs && (int)blockIdx.x >= __ldg(&probs[p + 1].cta0)) ++p;
  {
    const int* src = reinterpret_cast<const int*>(probs + p);
    int* dst = reinterpret_cast<int*>(&P);
    for (int i = threadIdx.x; i < (int)(sizeof(GemmProblem) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int local = blockIdx.x - P.cta0;
  // cluster mode: the splits of one tile are consecutive CTAs (one cluster)
  const int z = kCl ? local % P.splits : local / P.tiles;
  const int tile = kCl ? local / P.splits : local - z * P.tiles;
  const int m0 = (tile / P.tiles_n) * BM, n0 = (tile % P.tiles_n) * BN;
  if (!kAK) {
    for (int i = threadIdx.x; i < P.n_seg * BM; i += blockDim.x) {
      const int s = i / BM, r = i % BM;
      rowA[s][r] = m0 + r < P.M ? op_row(P.seg[s].A, m0 + r) : nullptr;
    }
  }
  if (kBN) {
    for (int i = threadIdx.x; i < P.n_seg * BN; i += blockDim.x) {
      const int s = i / BN, r = i % BN;
      rowB[s][r] = n0 + r < P.N ? op_row(P.seg[s].B, n0 + r) : nullptr;
    }
  }
  __syncthreads();

  int total_kt = 0;
  for (int s = 0; s < P.n_seg; ++s) total_kt += (P.seg[s].K + BK - 1) / BK;
  const int t0 = (int)((int64_t)total_kt * z / P.splits), t1 = (int)((int64_t)total_kt * (z + 1) / P.splits);

  using ALoad = TileLoad<kAK ? BK : BM, kAK ? BM : BK, C::kThreads>;
  using BLoad = TileLoad<kBN ? BN : BK, kBN ? BK : BN, C::kThreads>;
  ALoad la;
  BLoad lb;

  const int tx = threadIdx.x % (BN / TN), ty = threadIdx.x / (BN / TN);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  // k-tile t -> (segment, k0)
  auto fetch = [&](int t) {
    int s = 0;
    for (; s + 1 < P.n_seg; ++s) {
      const int nt = (P.seg[s].K + BK - 1) / BK;
      if (t < nt) break;
      t -= nt;
    }
    const GemmSeg& sg = P.seg[s];
    const int k0 = t * BK;
    if (kAK) la.load(sg.A, P.vec_a, k0, sg.K, m0, P.M);
    else la.load(sg.A, P.vec_a, m0, P.M, k0, sg.K, rowA[s]);
    if (kBN) lb.load(sg.B, P.vec_b, n0, P.N, k0, sg.K, rowB[s]);
    else lb.load(sg.B, P.vec_b, k0, sg.K, n0, P.N);
  };

  int buf = 0;
  if (t0 < t1) {
    fetch(t0);
    la.template store<!kAK, C::kApad>(As[0]);
    lb.template store<kBN, C::kBpad>(Bs[0]);
  }
  __syncthreads();
  for (int t = t0; t < t1; ++t) {
    if (t + 1 < t1) fetch(t + 1);
    const float* Ab = As[buf];
    const float* Bb = Bs[buf];
    // blocked summation: each k-tile accumulates into a fresh partial that is
    // then added to the running sum (error grows with K/BK + BK instead of K;
    // K reaches 10^4 for the output-layer dX)
    float tacc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) tacc[i][j] = 0.f;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float ra[TM], rb[TN];
#pragma unroll
      for (int g = 0; g < TM / 4; ++g) {
        const float4 x = *reinterpret_cast<const float4*>(Ab + k * C::kApad + g * (BM / (TM / 4)) + ty * 4);
        ra[g * 4 + 0] = x.x; ra[g * 4 + 1] = x.y; ra[g * 4 + 2] = x.z; ra[g * 4 + 3] = x.w;
      }
#pragma unroll
      for (int g = 0; g < TN / 4; ++g) {
        const float4 x = *reinterpret_cast<const float4*>(Bb + k * C::kBpad + g * (BN / (TN / 4)) + tx * 4);
        rb[g * 4 + 0] = x.x; rb[g * 4 + 1] = x.y; rb[g * 4 + 2] = x.z; rb[g * 4 + 3] = x.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) tacc[i][j] = fmaf(ra[i], rb[j], tacc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] += tacc[i][j];
    if (t + 1 < t1) {
      la.template store<!kAK, C::kApad>(As[buf ^ 1]);
      lb.template store<kBN, C::kBpad>(Bs[buf ^ 1]);
    }
    __syncthreads();
    buf ^= 1;
  }

  const bool has_bias = P.bias.rows != nullptr || P.bias.base != nullptr;
  if (kCl) {
    // partial tile -> own shared memory; after the cluster barrier CTA z
    // reduces rows [z*BM/S, (z+1)*BM/S) of the tile over the S partials read
    // through DSMEM (fixed split order: deterministic) and writes them out
    cgrp::cluster_group cl = cgrp::this_cluster();
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int g = 0; g < TN / 4; ++g) {
        const int lm = (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4);
        const int ln = g * (BN / (TN / 4)) + tx * 4;
        *reinterpret_cast<float4*>(red + lm * BN + ln) =
            make_float4(acc[i][g * 4], acc[i][g * 4 + 1], acc[i][g * 4 + 2], acc[i][g * 4 + 3]);
      }
    cl.sync();
    const int S = P.splits;
    const int rows = (BM + S - 1) / S;
    const int r0 = z * rows, r1 = min(BM, r0 + rows);
    for (int e = threadIdx.x; e < (r1 - r0) * BN; e += blockDim.x) {
      const int lm = r0 + e / BN, ln = e % BN;
      float s = 0.f;
      for (int q = 0; q < S; ++q) s += cl.map_shared_rank(red, q)[lm * BN + ln];
      const int m = m0 + lm, n = n0 + ln;
      if (m < P.M && n < P.N) {
        float* crow = const_cast<float*>(op_row(P.C, m));
        if (has_bias) s += op_row(P.bias, m)[n];
        if (P.accumulate) s += crow[n];
        crow[n] = s;
      }
    }
    cl.sync();  // keep every CTA's partial alive until all reads are done
    return;
  }
  if (P.splits > 1) {
    // partial tile -> workspace; the last split to arrive reduces in order
    float* part = work + P.work_off + (int64_t)z * ((int64_t)P.tiles * BM * BN) + (int64_t)tile * BM * BN;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int g = 0; g < TN / 4; ++g) {
        const int lm = (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4);
        const int ln = g * (BN / (TN / 4)) + tx * 4;
        __stcg(reinterpret_cast<float4*>(part + lm * BN + ln),
               make_float4(acc[i][g * 4], acc[i][g * 4 + 1], acc[i][g * 4 + 2], acc[i][g * 4 + 3]));
      }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int prev = atomicAdd(&counters[P.counter0 + tile], 1);
      s_last = prev == P.splits - 1;
      if (s_last) counters[P.counter0 + tile] = 0;  // reset for the next launch
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // splits outer, every element of the micro-tile in flight (float4 rows)
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
    for (int q = 0; q < P.splits; ++q) {
      const float* pq = work + P.work_off + (int64_t)q * ((int64_t)P.tiles * BM * BN) + (int64_t)tile * BM * BN;
      float4 v[TM][TN / 4];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int g = 0; g < TN / 4; ++g) {
          const int lm = (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4);
          const int ln = g * (BN / (TN / 4)) + tx * 4;
          v[i][g] = __ldcg(reinterpret_cast<const float4*>(pq + lm * BN + ln));
        }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int g = 0; g < TN / 4; ++g) {
          acc[i][g * 4 + 0] += v[i][g].x;
          acc[i][g * 4 + 1] += v[i][g].y;
          acc[i][g * 4 + 2] += v[i][g].z;
          acc[i][g * 4 + 3] += v[i][g].w;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4);
    if (m >= P.M) continue;
    float* crow = const_cast<float*>(op_row(P.C, m));
    const float* brow = has_bias ? op_row(P.bias, m) : nullptr;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + (j / 4) * (BN / (TN / 4)) + tx * 4 + (j % 4);
      if (n >= P.N) continue;
      float v = acc[i][j];
      if (brow) v += brow[n];
      if (P.accumulate) v += crow[n];
      crow[n] = v;
    }
  }
}

struct CfgInfo {
  int bm, bn, bk;
};
constexpr CfgInfo kCfg[4] = {{128, 128, 8}, {64, 64, 16}, {64, 32, 32}, {32, 32, 32}};

template <int BM, int BN, int BK, int TM, int TN, bool kAK, bool kBN>
void launch_one(const GemmLaunch& L, const GemmProblem* probs, float* work, int* counters, cudaStream_t s) {
  using C = Cfg<BM, BN, BK, TM, TN>;
  if (L.cluster > 0) {
    if constexpr (BM * BN <= 64 * 64) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(L.ctas);
      cfg.blockDim = dim3(C::kThreads);
      cfg.stream = s;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = L.cluster;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      cudaLaunchKernelEx(&cfg, gemm_group_kernel<BM, BN, BK, TM, TN, kAK, kBN, true>, probs, L.n_probs, work,
                         counters);
    }
    return;
  }
  launch_k(gemm_group_kernel<BM, BN, BK, TM, TN, kAK, kBN, false>, L.ctas, C::kThreads, 0, s, probs, L.n_probs, work,
                                                                                        counters);
}

template <int BM, int BN, int BK, int TM, int TN>
void launch_major(const GemmLaunch& L, const GemmProblem* probs, float* work, int* counters, cudaStream_t s) {
  if (L.a_kmajor && L.b_nmajor) launch_one<BM, BN, BK, TM, TN, true, true>(L, probs, work, counters, s);
  else if (L.a_kmajor) launch_one<BM, BN, BK, TM, TN, true, false>(L, probs, work, counters, s);
  else if (L.b_nmajor) launch_one<BM, BN, BK, TM, TN, false, true>(L, probs, work, counters, s);
  else launch_one<BM, BN, BK, TM, TN, false, false>(L, probs, work, counters, s);
}

bool base_vec_ok(const Operand& o) {
  if (o.rows) return o.rows_aligned != 0;
  return (reinterpret_cast<uintptr_t>(o.base) % 16 == 0) && (o.ld % 4 == 0);
}

}  // namespace

GemmLaunch gemm_plan(std::vector<GemmProblem>& probs, bool a_kmajor, bool b_nmajor, int64_t work_cap_floats,
                     int counter_cap) {
  GemmLaunch L{};
  L.a_kmajor = a_kmajor;
  L.b_nmajor = b_nmajor;
  L.n_probs = (int)probs.size();
  int max_m = 0;
  double flops = 0;
  for (auto& p : probs) {
    max_m = std::max(max_m, p.M);
    int64_t k = 0;
    for (int s = 0; s < p.n_seg; ++s) k += p.seg[s].K;
    flops += 2.0 * p.M * p.N * (double)k;
  }
  // tile shape: skinny problems (the recurrent steps, M = minibatch) get
  // 64x32 tiles; big ones 128x128; the rest 64x64
  int64_t t128 = 0;
  for (auto& p : probs) t128 += (int64_t)((p.M + 127) / 128) * ((p.N + 127) / 128);
  if (!a_kmajor && max_m <= 64) L.cfg = 2;
  else if (t128 >= 120) L.cfg = 0;
  else if (max_m <= 32 && !a_kmajor) L.cfg = 3;
  else L.cfg = 1;
  const CfgInfo c = kCfg[L.cfg];
  const int threads = L.cfg == 3 ? 64 : (L.cfg == 2 ? 128 : 256);
  int64_t tiles_all = 0;
  for (auto& p : probs) {
    p.tiles_n = (p.N + c.bn - 1) / c.bn;
    p.tiles = ((p.M + c.bm - 1) / c.bm) * p.tiles_n;
    tiles_all += p.tiles;
  }
  // split-K so that roughly two waves of 256-thread-equivalents are in flight
  const int64_t target = (int64_t)148 * 2 * 256 / threads;
  // smaller tiles: one uniform split count per launch, the splits of a tile
  // forming a thread-block cluster (DSMEM reduction, no global partials)
  L.cluster = 0;
  if (L.cfg != 0) {
    int min_kt = 1 << 30;
    for (auto& p : probs) {
      int kt = 0;
      for (int s = 0; s < p.n_seg; ++s) kt += (p.seg[s].K + c.bk - 1) / c.bk;
      min_kt = std::min(min_kt, kt);
    }
    int S = (int)std::min<int64_t>((target + tiles_all - 1) / tiles_all, 8);
    S = std::max(1, std::min(S, std::max(1, min_kt)));
    if (S > 1) L.cluster = S;
  }
  int64_t cta = 0, counter = 0, woff = 0;
  for (auto& p : probs) {
    int kt = 0;
    for (int s = 0; s < p.n_seg; ++s) kt += (p.seg[s].K + c.bk - 1) / c.bk;
    int splits = 1;
    if (L.cluster > 0) {
      splits = L.cluster;
    } else if (tiles_all < target && kt >= 4) {
      splits = (int)std::min<int64_t>((target + tiles_all - 1) / tiles_all, kt / 2);
      splits = std::max(1, std::min(splits, 8));
    }
    const int64_t part = (int64_t)splits * p.tiles * c.bm * c.bn;
    if (L.cluster == 0 && splits > 1 && (woff + part > work_cap_floats || counter + p.tiles > counter_cap)) splits = 1;
    p.splits = splits;
    p.cta0 = (int)cta;
    p.counter0 = (int)counter;
    p.work_off = woff;
    if (splits > 1 && L.cluster == 0) {
      woff += part;
      counter += p.tiles;
    }
    cta += (int64_t)p.tiles * splits;
    // vectorised loads need 16B-aligned rows and contiguous extents % 4
    bool va = true, vb = true;
    for (int s = 0; s < p.n_seg; ++s) {
      const GemmSeg& sg = p.seg[s];
      va = va && base_vec_ok(sg.A) && ((a_kmajor ? p.M : sg.K) % 4 == 0);
      vb = vb && base_vec_ok(sg.B) && ((b_nmajor ? sg.K : p.N) % 4 == 0);
    }
    p.vec_a = va;
    p.vec_b = vb;
  }
  L.ctas = (int)cta;
  L.work_floats = woff;
  L.flops = flops;
  return L;
}

int launch_gemm_group(const GemmLaunch& L, const GemmProblem* probs_dev, float* work, int* counters,
                      cudaStream_t s) {
  if (L.ctas <= 0) return 0;
  switch (L.cfg) {
    case 0: launch_major<128, 128, 8, 8, 8>(L, probs_dev, work, counters, s); break;
    case 1: launch_major<64, 64, 16, 4, 4>(L, probs_dev, work, counters, s); break;
    case 2: launch_major<64, 32, 32, 4, 4>(L, probs_dev, work, counters, s); break;
    default: launch_major<32, 32, 32, 4, 4>(L, probs_dev, work, counters, s); break;
  }
  return 1;
}

}  // namespace dg
