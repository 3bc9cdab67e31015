// Persistent LSTM recurrence kernels (sm_100a, fp32).
//
// The reference evaluates an LSTM layer-step as 13 graph nodes
// (builders.py:92-101: gates = affine(b, Wx, x, Wh, h); i,f,o = logistic(
// pick_range), g = tanh(pick_range); c = f*c_prev + i*g; h = o*tanh(c)) and
// interprets them one node at a time (graph.py:115-164).  The executor's
// planner recognises chains of such steps that share (Wx, Wh, b) and feed
// h_t / c_t into step t+1, stacks chains whose inputs are another chain's
// outputs (x^l_t = h^{l-1}_t), and runs the whole recurrence of a stack in ONE
// launch per direction:
//
//   * one CTA per (batch slice of BS rows, block of 16 hidden units) per
//     chain; the CTA keeps its slice of the weights resident in shared memory
//     for every step (forward: the 64 gate columns of its units over
//     [Wx | Wh]; backward: the 16 columns of Wh^T and of the consumer
//     chain's Wx^T), so weights are read from HBM once per launch;
//   * batch rows never interact in an LSTM, so a CTA only waits for the CTAs
//     of its own batch slice: per-(chain, slice, step) arrival counters in
//     global memory (release: __threadfence + atomicAdd; acquire:
//     ld.acquire.gpu), a stacked chain waits for its producer chain's step t
//     only -> the layers run as a wavefront without a grid-wide barrier;
//   * every node of the pattern keeps its own value and gradient slot (same
//     arithmetic as cell_fwd_kernel / cell_bwd_kernel in kernels.cu).
//
// Gradient flow in the backward kernel (per CTA, rows R, units U):
//   dh_t[R,U] = slot(h_t) (contributions of consumers outside the stack, all
//               complete before the launch) + rec_t + cons_t
//   rec_t     = sum_j Wh[j,U] dG_{t+1}[R,j]          (own chain, step t+1)
//   cons_t    = sum_j Wx'[j,U] dG'_t[R,j]            (consumer chain, step t)
//   then the cell backward writes every internal gradient, dG_t[R, own
//   columns] and c_{t-1}'s gradient.  Gradients of external inputs (x_t of
//   the bottom chain, h_{-1}) and the weight / bias gradients are batched
//   GEMMs / column sums planned by the executor after this launch; a
//   batch-1 (broadcast) c_{-1} gets its batch sum from rnn_c0_kernel.
//
// Co-residency: launched with cudaLaunchCooperativeKernel (one CTA per SM at
// most, grid <= SM count checked by the planner), so spinning CTAs can never
// starve a producer.  A bounded spin traps instead of hanging the GPU.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "kernels.cuh"

namespace dg {

bool rnn_trace_enabled();

namespace {

constexpr int kRT = 256;  // threads per CTA
constexpr int kU = kRnnUnits;
constexpr int kCU = 4 * kU;  // gate columns per CTA
constexpr int kSmCountTrace = 148;

__device__ __forceinline__ float sigmoid_ref(float x) {
  x = fminf(fmaxf(x, -60.f), 60.f);  // ops.py:78-83
  return 1.f / (1.f + expf(-x));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_count(const int* p, int target) {
  if (ld_acquire(p) >= target) return;
  unsigned spins = 0;
  while (ld_acquire(p) < target) {
    __nanosleep(32);
    if (++spins > (1u << 24)) __trap();  // a missing producer: fail, never hang
  }
}

__device__ __forceinline__ void arrive(int* p) {
  __threadfence();
  atomicAdd(p, 1);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// optional timeline (DG_RNN_TRACE=1): per CTA [0] start, [1] weights resident,
// [2 + t] arrival of step t (forward order for both kernels), globaltimer ns
constexpr int kTraceSlots = 256;
__device__ unsigned long long g_rnn_trace[2][kSmCountTrace][kTraceSlots];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace(int kind, int slot) {
  if (slot < kTraceSlots && blockIdx.x < kSmCountTrace) g_rnn_trace[kind][blockIdx.x][slot] = gtimer();
}

// barrier among the 256 compute threads (named barrier 1); the cluster
// kernels add a signalling warp that must not join these
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ int chain_of(const RnnArgs& a, int cta) {
  int ci = 0;
  while (ci + 1 < a.n_chains && cta >= a.ch[ci + 1].cta0) ++ci;
  return ci;
}

// gate column of a lane's c-th accumulator (lane column group lc of LC):
// 4-wide chunks interleaved across lanes so a quarter-warp's float4 accesses
// cover 128 contiguous bytes (no bank conflicts on the partial-sum stores)
template <int LC, int TC>
__device__ __forceinline__ int lane_col(int lc, int c) {
  if constexpr (TC >= 4) return (c >> 2) * (LC * 4) + lc * 4 + (c & 3);
  else return lc * TC + c;
}

// slots per step (CellSlots with m = 1, kernels.cu) + x_t + h_{t-1}
enum : int {
  S_G = 0, S_CP = 1, S_PI = 2, S_PF = 3, S_PO = 4, S_PG = 5, S_AI = 6, S_AF = 7, S_AO = 8, S_AG = 9,
  S_IG = 10, S_FC = 11, S_C = 12, S_TC = 13, S_H = 14, S_X = 15, S_HP = 16
};

// ---------------------------------------------------------------- forward
// Shared-memory step table: the 17 node pointers (+ batch-1 flags) of step t
// are prefetched one step ahead by warp 1 into a double buffer, so the step's
// critical path never waits on a pointer load.
struct StepPtrs {
  const float* p[kRnnSlots];
  int b1;
};

template <int BS>
__global__ void __launch_bounds__(kRT, 1) rnn_fwd_kernel(const __grid_constant__ RnnArgs a) {
  pdl_prologue();
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ StepPtrs sp[2];
  const int ci = chain_of(a, blockIdx.x);
  const RnnChain C = a.ch[ci];  // register copy (dynamic-index constant loads are slow)
  const int local = blockIdx.x - C.cta0;
  const int s = local / C.n_u, ub = local - (local / C.n_u) * C.n_u;
  const int b0 = s * BS, j0 = ub * kU;
  const int K = C.K_in + C.H;
  float* Ws = sm;                          // [K][kCU]
  const int KP = K + 4;                    // padded row stride (16B rows, no bank conflicts)
  float* inS = Ws + (size_t)K * kCU;       // [BS][K+4]
  float* part = inS + (size_t)BS * KP;     // [8][BS][kCU]
  float* bias = part + 8 * BS * kCU;       // [kCU]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int goff[4] = {C.off_i, C.off_f, C.off_o, C.off_g};
  if (a.trace && tid == 0) trace(0, 0);

  // resident weight slice: column c = gate * 16 + jj  <->  G row goff[gate] + j0 + jj
  if (a.vec) {
    for (int idx = tid; idx < K * (kCU / 4); idx += kRT) {
      const int k = idx / (kCU / 4), q = idx - k * (kCU / 4);
      const int gate = q / (kU / 4), j = j0 + 4 * (q - gate * (kU / 4));
      float* dst = Ws + (size_t)k * kCU + 4 * q;
      if (j < C.H) {
        const int64_t row = goff[gate] + j;
        cp_async16(dst, k < C.K_in ? C.Wx + row + (int64_t)k * C.gw : C.Wh + row + (int64_t)(k - C.K_in) * C.gw);
      } else {
        *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  } else {
    for (int idx = tid; idx < K * kCU; idx += kRT) {
      const int k = idx / kCU, c = idx - (idx / kCU) * kCU;
      const int gate = c / kU, j = j0 + (c - gate * kU);
      float w = 0.f;
      if (j < C.H) {
        const int64_t row = goff[gate] + j;
        w = k < C.K_in ? C.Wx[row + (int64_t)k * C.gw] : C.Wh[row + (int64_t)(k - C.K_in) * C.gw];
      }
      Ws[(size_t)k * kCU + c] = w;
    }
  }
  if (tid < kCU) {
    const int gate = tid / kU, j = j0 + (tid - gate * kU);
    bias[tid] = j < C.H ? C.bias[goff[gate] + j] : 0.f;
  }
  if (tid < kRnnSlots) sp[0].p[tid] = C.val[tid];
  if (tid == kRnnSlots) sp[0].b1 = C.b1[0];
  cp_async_wait_all();
  __syncthreads();
  if (a.trace && tid == 0) trace(0, 1);

  int* my_flags = a.flags + C.flag0 + s * C.T;
  const int* src_flags = nullptr;
  int src_need = 0;
  if (C.src >= 0) {
    const RnnChain& P = a.ch[C.src];
    src_flags = a.flags + P.flag0 + s * P.T;
    src_need = P.n_u;
  }

  constexpr int LB = BS < 4 ? BS : 4;
  constexpr int TB = BS / LB;
  constexpr int LC = 32 / LB;
  constexpr int TC = kCU / LC;
  const int lb = lane / LC, lc = lane - (lane / LC) * LC;
  const int cb = tid / kU, cj = tid - (tid / kU) * kU;  // cell thread: (row, unit)
  const int crow = b0 + cb, cjj = j0 + cj;
  const bool cell_mine = cb < BS && crow < C.B && cjj < C.H;
  float c_carry = 0.f;  // c_{t-1} of this thread's (row, unit), produced by itself

  // stage columns [k_lo, k_hi) of this slice's [x_t | h_{t-1}] rows (L2 -> smem, bypassing L1)
  auto stage = [&](const float* src, int64_t ld, bool b1, int k_lo, int k_hi) {
    if (a.vec) {
      const int w4 = (k_hi - k_lo) >> 2;
      for (int idx = tid; idx < BS * w4; idx += kRT) {
        const int b = idx / w4, q = idx - (idx / w4) * w4;
        const int row = b0 + b;
        float* dst = inS + (size_t)b * KP + k_lo + 4 * q;
        if (row < C.B) cp_async16(dst, src + (b1 ? 0 : (int64_t)row * ld) + 4 * q);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cp_async_wait_all();
    } else {
      const int w = k_hi - k_lo;
      for (int idx0 = tid; idx0 < BS * w; idx0 += 4 * kRT) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = idx0 + q * kRT;
          const int b = idx / w, k = idx - (idx / w) * w;
          v[q] = (idx < BS * w && b0 + b < C.B) ? __ldcg(src + (b1 ? 0 : (int64_t)(b0 + b) * ld) + k) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = idx0 + q * kRT;
          if (idx < BS * w) inS[(size_t)(idx / w) * KP + k_lo + (idx - (idx / w) * w)] = v[q];
        }
      }
    }
  };
  float acc[TB][TC];
  // acc += rows[:, k_lo:k_hi] W[k_lo:k_hi, :] over this warp's share of the range
  auto fma_range = [&](int k_lo, int k_hi) {
    const int per = (k_hi - k_lo + 7) / 8;
    const int kb = k_lo + warp * per, ke = min(k_hi, kb + per);
#pragma unroll 4
    for (int k = kb; k < ke; ++k) {
      float xa[TB], wv[TC];
#pragma unroll
      for (int i = 0; i < TB; ++i) xa[i] = inS[(size_t)(i * LB + lb) * KP + k];
#pragma unroll
      for (int c = 0; c < TC; ++c) wv[c] = Ws[(size_t)k * kCU + lane_col<LC, TC>(lc, c)];
#pragma unroll
      for (int i = 0; i < TB; ++i)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[i][c] = fmaf(xa[i], wv[c], acc[i][c]);
    }
  };

  for (int t = 0; t < C.T; ++t) {
    const StepPtrs& P = sp[t & 1];
    // prefetch step t+1's pointers (consumed after the next barrier)
    const float* nxt = nullptr;
    int nxt_b1 = 0;
    if (warp == 1 && t + 1 < C.T) {
      if (lane < kRnnSlots) nxt = C.val[(size_t)(t + 1) * kRnnSlots + lane];
      if (lane == kRnnSlots) nxt_b1 = C.b1[t + 1];
    }
    const int fl = P.b1;
    if (t == 0 && cell_mine) c_carry = __ldcg(P.p[S_CP] + ((fl & 4) ? cjj : (int64_t)crow * C.H + cjj));
    // gx mode: the G slot already holds b + Wx x_t (batched tensor-core GEMM
    // before this launch); read it ahead of the waits
    float gx[4] = {0.f, 0.f, 0.f, 0.f};
    if (a.gx && cell_mine) {
      const float* Gr = P.p[S_G] + (int64_t)crow * C.gw;
      gx[0] = Gr[C.off_i + cjj];
      gx[1] = Gr[C.off_f + cjj];
      gx[2] = Gr[C.off_o + cjj];
      gx[3] = Gr[C.off_g + cjj];
    }
#pragma unroll
    for (int i = 0; i < TB; ++i)
#pragma unroll
      for (int c = 0; c < TC; ++c) acc[i][c] = 0.f;
    // input part: needs only x_t (external, or the producer chain's step t),
    // so it overlaps the arrival of this chain's step t-1
    if (C.K_in > 0) {
      if (tid == 0 && src_flags) wait_count(src_flags + t, src_need);
      __syncthreads();
      stage(P.p[S_X], C.K_in, (fl & 1) != 0, 0, C.K_in);
      __syncthreads();
      fma_range(0, C.K_in);
    }
    // recurrent part: h_{t-1} of every unit block of this batch slice
    if (tid == 0 && t > 0) wait_count(my_flags + t - 1, C.n_u);
    __syncthreads();
    stage(P.p[S_HP], C.H, (fl & 2) != 0, C.K_in, K);
    __syncthreads();
    fma_range(C.K_in, K);
#pragma unroll
    for (int i = 0; i < TB; ++i)
#pragma unroll
      for (int c = 0; c < TC; ++c) part[(warp * BS + i * LB + lb) * kCU + lane_col<LC, TC>(lc, c)] = acc[i][c];
    __syncthreads();
    float x4[4] = {0.f, 0.f, 0.f, 0.f}, ai = 0.f, af = 0.f, ao = 0.f, ag = 0.f, ig = 0.f, p = 0.f, c = 0.f, tc = 0.f;
    const int64_t r = (int64_t)crow * C.H + cjj;
    if (cell_mine) {
#pragma unroll
      for (int gate = 0; gate < 4; ++gate) {
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) sum += part[(w * BS + cb) * kCU + gate * kU + cj];
        x4[gate] = (a.gx ? gx[gate] : bias[gate * kU + cj]) + sum;
      }
      ai = sigmoid_ref(x4[0]);
      af = sigmoid_ref(x4[1]);
      ao = sigmoid_ref(x4[2]);
      ag = tanhf(x4[3]);
      ig = ai * ag;
      p = af * c_carry;
      c = ig + p;
      c_carry = c;
      tc = tanhf(c);
      // the critical output (read by the other CTAs of the slice) first
      const_cast<float*>(P.p[S_H])[r] = ao * tc;
    }
    if (warp == 1 && t + 1 < C.T) {
      if (lane < kRnnSlots) sp[(t + 1) & 1].p[lane] = nxt;
      if (lane == kRnnSlots) sp[(t + 1) & 1].b1 = nxt_b1;
    }
    __syncthreads();
    if (tid == 0) {
      arrive(my_flags + t);
      if (a.trace) trace(0, 2 + t);
    }
    if (cell_mine) {
      // every other node of the step keeps its value slot (off the critical path)
      float* G = const_cast<float*>(P.p[S_G]) + (int64_t)crow * C.gw;
      G[C.off_i + cjj] = x4[0];
      G[C.off_f + cjj] = x4[1];
      G[C.off_o + cjj] = x4[2];
      G[C.off_g + cjj] = x4[3];
      auto W = [&](int slot, float v) { const_cast<float*>(P.p[slot])[r] = v; };
      W(S_PI, x4[0]);
      W(S_PF, x4[1]);
      W(S_PO, x4[2]);
      W(S_PG, x4[3]);
      W(S_AI, ai);
      W(S_AF, af);
      W(S_AO, ao);
      W(S_AG, ag);
      W(S_IG, ig);
      W(S_FC, p);
      W(S_C, c);
      W(S_TC, tc);
    }
  }
}

// ---------------------------------------------------------------- backward
// out[BS][16] = sum_j dG[R, j] * WT[j][16]: the rows' gate gradients are staged
// through shared memory (row stride CJ+4) in chunks of CJ columns; warps split
// j, lanes tile (rows x units); partials are reduced in fixed order.
template <int BS>
__device__ __forceinline__ float rows_times_wt(const float* dG, int gw, int B, int b0, const float* WT,
                                               float* dGs, int CJ, float* part, bool vec) {
  constexpr int LB = BS < 8 ? BS : 8;
  constexpr int TB = BS / LB;
  constexpr int LC = (32 / LB) < kU ? (32 / LB) : kU;
  constexpr int TC = kU / LC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lb = lane / LC, lc = lane - (lane / LC) * LC;
  const bool active = lb < LB;
  float acc[TB][TC];
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[i][c] = 0.f;
  const int CP = CJ + 4;  // padded row stride
  for (int jc = 0; jc < gw; jc += CJ) {
    const int cj = min(CJ, gw - jc);
    if (vec) {
      const int c4 = cj >> 2;
      for (int idx = tid; idx < BS * c4; idx += kRT) {
        const int b = idx / c4, q = idx - (idx / c4) * c4;
        const int row = b0 + b;
        float* dst = dGs + (size_t)b * CP + 4 * q;
        if (row < B) cp_async16(dst, dG + (int64_t)row * gw + jc + 4 * q);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cp_async_wait_all();
    } else {
      for (int idx0 = tid; idx0 < BS * cj; idx0 += 4 * kRT) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = idx0 + q * kRT;
          const int b = idx / cj, jl = idx - (idx / cj) * cj;
          v[q] = (idx < BS * cj && b0 + b < B) ? __ldcg(dG + (int64_t)(b0 + b) * gw + jc + jl) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = idx0 + q * kRT;
          if (idx < BS * cj) dGs[(size_t)(idx / cj) * CP + (idx - (idx / cj) * cj)] = v[q];
        }
      }
    }
    csync();
    const int per = (cj + 7) / 8;
    const int jb = warp * per, je = min(cj, jb + per);
    if (active) {
#pragma unroll 4
      for (int jl = jb; jl < je; ++jl) {
        float xa[TB], wv[TC];
#pragma unroll
        for (int i = 0; i < TB; ++i) xa[i] = dGs[(size_t)(i * LB + lb) * CP + jl];
#pragma unroll
        for (int c = 0; c < TC; ++c) wv[c] = WT[(size_t)(jc + jl) * kU + lc * TC + c];
#pragma unroll
        for (int i = 0; i < TB; ++i)
#pragma unroll
          for (int c = 0; c < TC; ++c) acc[i][c] = fmaf(xa[i], wv[c], acc[i][c]);
      }
    }
    csync();
  }
  if (active) {
#pragma unroll
    for (int i = 0; i < TB; ++i)
#pragma unroll
      for (int c = 0; c < TC; ++c) part[(warp * BS + i * LB + lb) * kU + lc * TC + c] = acc[i][c];
  }
  csync();
  const int cb = tid / kU, cu = tid - (tid / kU) * kU;
  float sum = 0.f;
  if (cb < BS) {
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += part[(w * BS + cb) * kU + cu];
  }
  csync();
  return sum;
}

struct StepPtrs2 {
  const float* v[kRnnSlots];
  float* d[kRnnSlots];
  int b1;
};

template <int BS>
__global__ void __launch_bounds__(kRT, 1) rnn_bwd_kernel(const __grid_constant__ RnnArgs a) {
  pdl_prologue();
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ StepPtrs2 sp[2];
  const int ci = chain_of(a, blockIdx.x);
  const RnnChain C = a.ch[ci];  // register copy (dynamic-index constant loads are slow)
  const int local = blockIdx.x - C.cta0;
  const int s = local / C.n_u, ub = local - (local / C.n_u) * C.n_u;
  const int b0 = s * BS, j0 = ub * kU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RnnChain* Cc = C.cons >= 0 ? &a.ch[C.cons] : nullptr;
  const int gw_c = Cc ? Cc->gw : 0;
  if (a.trace && tid == 0) trace(1, 0);
  float* WhT = sm;                              // [gw][16]
  float* WcT = WhT + (size_t)C.gw * kU;         // [gw_c][16]
  float* dGs = WcT + (size_t)gw_c * kU;         // [BS][CJ+4]
  float* part = dGs + (size_t)(a.cj + 4) * BS;  // [8][BS][16]

  // W^T slices: WT[j][u] = W[j + (j0+u) * gw]   (column j0+u of W, contiguous in j)
  for (int idx = tid; idx < C.gw * kU; idx += kRT) {
    const int u = idx / C.gw, j = idx - (idx / C.gw) * C.gw;
    float* dst = WhT + (size_t)j * kU + u;
    if (j0 + u < C.H) cp_async4(dst, C.Wh + j + (int64_t)(j0 + u) * C.gw);
    else *dst = 0.f;
  }
  if (Cc) {
    for (int idx = tid; idx < gw_c * kU; idx += kRT) {
      const int u = idx / gw_c, j = idx - (idx / gw_c) * gw_c;
      float* dst = WcT + (size_t)j * kU + u;
      if (j0 + u < C.H) cp_async4(dst, Cc->Wx + j + (int64_t)(j0 + u) * gw_c);
      else *dst = 0.f;
    }
  }
  {
    const int t = C.T - 1;
    if (tid < kRnnSlots) sp[t & 1].v[tid] = C.val[(size_t)t * kRnnSlots + tid];
    if (tid >= 32 && tid < 32 + kRnnSlots) sp[t & 1].d[tid - 32] = C.grad[(size_t)t * kRnnSlots + tid - 32];
    if (tid == 64) sp[t & 1].b1 = C.b1[t];
  }
  cp_async_wait_all();
  __syncthreads();
  if (a.trace && tid == 0) trace(1, 1);

  int* my_flags = a.flags + C.flag0 + s * C.T;
  const int* cons_flags = Cc ? a.flags + Cc->flag0 + s * Cc->T : nullptr;
  const int cb = tid / kU, cj = tid - (tid / kU) * kU;
  const int row = b0 + cb, j = j0 + cj;
  const bool mine = cb < BS && row < C.B && j < C.H;
  const int64_t r = (int64_t)row * C.H + j;
  float rec = 0.f;       // dh_t from step t+1 of this chain
  float cons = 0.f;      // dh_t from the consumer chain's step t
  float dc_carry = 0.f;  // dc_t contribution of step t+1 (f_{t+1} * dc_{t+1})
  // forward values and external gradient contributions of step t's cell: all
  // independent of other CTAs, loaded ahead of the waits
  float ao = 0.f, ai = 0.f, ag = 0.f, tc = 0.f, af = 0.f, ck = 0.f, gh_ext = 0.f, gc_ext = 0.f;
  auto load_cell = [&](const StepPtrs2& P) {
    if (!mine) return;
    const bool cb1 = (P.b1 & 4) != 0;
    ao = P.v[S_AO][r];
    ai = P.v[S_AI][r];
    ag = P.v[S_AG][r];
    tc = P.v[S_TC][r];
    af = P.v[S_AF][r];
    ck = P.v[S_CP][cb1 ? j : r];
    gh_ext = P.d[S_H][r];
    gc_ext = P.d[S_C][r];
  };
  load_cell(sp[(C.T - 1) & 1]);
  if (Cc) {
    if (tid == 0) wait_count(cons_flags + C.T - 1, Cc->n_u);
    __syncthreads();
    cons = rows_times_wt<BS>(Cc->grad[(size_t)(C.T - 1) * kRnnSlots + S_G], gw_c, C.B, b0, WcT, dGs, a.cj, part,
                             a.vec);
  }

  for (int t = C.T - 1; t >= 0; --t) {
    const StepPtrs2& P = sp[t & 1];
    // prefetch step t-1's pointers (published to smem before the next barrier)
    const float* nv = nullptr;
    float* nd = nullptr;
    int nb1 = 0;
    if (warp == 1 && t > 0) {
      if (lane < kRnnSlots) {
        nv = C.val[(size_t)(t - 1) * kRnnSlots + lane];
        nd = C.grad[(size_t)(t - 1) * kRnnSlots + lane];
      }
      if (lane == kRnnSlots) nb1 = C.b1[t - 1];
    }
    const bool cb1 = (P.b1 & 4) != 0;
    float gh = 0.f, d_tc = 0.f, d_o = 0.f, dc = 0.f, d_i = 0.f, d_g = 0.f, dpi = 0.f, dpo = 0.f, dpg = 0.f;
    float d_f = 0.f, dpf = 0.f;
    if (mine) {
      // cell backward; the gate gradients (read by the other CTAs of the
      // slice) are stored first.  Internal slots have this cell as their
      // only consumer: written, not accumulated.
      gh = gh_ext + rec + cons;
      d_tc = gh * ao;
      d_o = gh * tc;
      dc = (gc_ext + dc_carry) + (1.f - tc * tc) * d_tc;
      d_i = dc * ag;
      d_g = dc * ai;
      dpi = ai * (1.f - ai) * d_i;
      dpo = ao * (1.f - ao) * d_o;
      dpg = (1.f - ag * ag) * d_g;
      d_f = dc * ck;
      dpf = af * (1.f - af) * d_f;
      float* dG = P.d[S_G] + (int64_t)row * C.gw;
      dG[C.off_i + j] = dpi;
      dG[C.off_o + j] = dpo;
      dG[C.off_g + j] = dpg;
      dG[C.off_f + j] = dpf;
      dc_carry = dc * af;
    }
    if (warp == 1 && t > 0) {
      if (lane < kRnnSlots) {
        sp[(t - 1) & 1].v[lane] = nv;
        sp[(t - 1) & 1].d[lane] = nd;
      }
      if (lane == kRnnSlots) sp[(t - 1) & 1].b1 = nb1;
    }
    __syncthreads();
    if (tid == 0) {
      arrive(my_flags + t);
      if (a.trace) trace(1, 2 + t);
    }
    if (mine) {
      float* const* D = P.d;
      D[S_H][r] = gh;
      D[S_TC][r] = d_tc;
      D[S_AO][r] = d_o;
      D[S_C][r] = dc;
      D[S_IG][r] = dc;
      D[S_AI][r] = d_i;
      D[S_AG][r] = d_g;
      D[S_PI][r] = dpi;
      D[S_PO][r] = dpo;
      D[S_PG][r] = dpg;
      D[S_FC][r] = dc;
      D[S_AF][r] = d_f;
      D[S_PF][r] = dpf;
      // c_{-1}: external state (batch-1 broadcast: rnn_c0_kernel sums it)
      if (t == 0 && !cb1) D[S_CP][r] += dc_carry;
    }
    if (t > 0) {
      load_cell(sp[(t - 1) & 1]);
      // consumer chain's step t-1 (runs ahead of this chain): off the critical path
      if (Cc) {
        if (tid == 0) wait_count(cons_flags + t - 1, Cc->n_u);
        __syncthreads();
        cons = rows_times_wt<BS>(Cc->grad[(size_t)(t - 1) * kRnnSlots + S_G], gw_c, C.B, b0, WcT, dGs, a.cj, part,
                                 a.vec);
      }
      if (tid == 0) wait_count(my_flags + t, C.n_u);
      __syncthreads();
      rec = rows_times_wt<BS>(P.d[S_G], C.gw, C.B, b0, WhT, dGs, a.cj, part, a.vec);
    }
  }
}

// ====================================================================
// Cluster variants: one thread-block cluster per (chain, batch slice) -- the
// n_u CTAs that exchange h_t (forward) / dG_t (backward) every step.  The
// exchange goes through distributed shared memory instead of L2:
//   forward : each CTA pushes its (rows x 16 units) slice of h_t into every
//             peer's double-buffered h operand block (st.shared::cluster) and
//             arrives on the peers' mbarrier (release.cluster); a CTA waits on
//             its own mbarrier (acquire.cluster) before the recurrent GEMM;
//   backward: reduce-scatter -- each CTA multiplies its own 64 gate columns of
//             dG_t by the matching rows of Wh (all units) and pushes the
//             partial dh_{t-1} of every peer's 16 units into that peer's slot;
//             the owner sums the n_u slots in rank order (deterministic).
// Cross-chain dependencies (stacked layers) stay on global arrival counters,
// published by a dedicated signalling warp (warp 8) so the fence never sits
// on the compute warps' critical path.
constexpr int kClThreads = kRT + 32;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_init_cl(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_addr(b);
  unsigned spins = 0;
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (!done && ++spins > (1u << 24)) __trap();
  }
}
// remote store that completes `bytes` of a transaction on the destination
// CTA's mbarrier: no fence / barrier needed on the producer side
__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(remote_addr), "f"(v),
               "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, float4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote_addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t remote_addr, float2 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(remote_addr),
               "f"(v.x), "f"(v.y), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 3xTF32 legacy-MMA tile op: acc(16 x 8) += A(16 x 8) B(8 x 8); a/b hold fp32
// bit patterns, the residuals lo = x - tf32(x) make A_hi B_hi + A_hi B_lo +
// A_lo B_hi (fp32-accurate products, as the tcgen05 GEMMs)
// Splits for 3xTF32.  Resident weight fragments (split once per launch):
// both parts rounded to nearest (cvt.rna, kernels.cuh), so lo has either
// sign.  Per-step operands (h_{t-1} forward, dG_t backward, split inside the
// k-loop by every warp): hi truncated, lo = x - hi exact.  The k-loop is
// bound by the legacy tensor pipe and shared-memory bandwidth together
// (tools/rnn_step_probe.cu), so every ALU op per element shows: rounding hi
// there costs +14% on the forward step (cvt.rna on both parts +17%) for no
// measurable change of the parity ratios (r02 A/B, tools/gpu/gpu_ab_src.sh).
__device__ __forceinline__ uint32_t tf32_hi(float x) { return tf32_rn_hi(x); }
__device__ __forceinline__ uint32_t tf32_lo(float x) { return tf32_rn_lo(x); }
__device__ __forceinline__ uint32_t step_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }
__device__ __forceinline__ uint32_t step_lo(float x, uint32_t hi) { return __float_as_uint(x - __uint_as_float(hi)); }
__device__ __forceinline__ void mma_1688(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Forward recurrence (gx mode: G slots hold b + Wx x_t): per step the CTA
// computes G_rec[16 rows x 64 gate columns] = h_{t-1}[rows, :] Wh^T[:, cols]
// on the tensor cores (warp w owns columns 8w..8w+7, 3xTF32 mma.sync over K =
// H), adds Gx, runs the cell and pushes its 16-unit slice of h_t to the
// cluster through distributed shared memory.
template <int BS>
__global__ void __launch_bounds__(kClThreads, 1) rnn_fwd_cl_kernel(const __grid_constant__ RnnArgs a) {
  // (pdl_prologue after the weight staging below)
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ StepPtrs sp[2];
  __shared__ __align__(8) uint64_t h_full[2];  // h_u lands in buffer u&1 (st.async transactions)
  const int ci = chain_of(a, blockIdx.x);
  const RnnChain C = a.ch[ci];  // register copy (dynamic-index constant loads are slow)
  const int local = blockIdx.x - C.cta0;
  const int s = local / C.n_u, ub = local - (local / C.n_u) * C.n_u;
  const int b0 = s * BS, j0 = ub * kU;
  const int KS = (C.H + 7) / 8;                 // k-steps of 8 over the recurrent input
  const int HP = 8 * KS + 4;                    // padded row stride: k-steps never leave the row
  float4* Bf = reinterpret_cast<float4*>(sm);   // [KS][8 warps][32 lanes] weight fragments (hi, lo)
  float* hS = sm + (size_t)KS * 8 * 32 * 4;     // [2][BS][HP]
  float* gS = hS + 2 * (size_t)BS * HP;         // [BS][64 + 4] recurrent gate sums
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int goff[4] = {C.off_i, C.off_f, C.off_o, C.off_g};
  const int g8 = lane >> 2, t4 = lane & 3;      // mma fragment coordinates
  if (a.trace && tid == 0) trace(0, 0);
  // h_{-1} source (flags, pointer): loaded first so its latency overlaps the
  // weight staging below
  const int fl_hp = C.b1[0];
  const float* Hp0 = C.val[S_HP];

  if (warp < 8) {
    // weight fragments: warp w, k-step q, lane (g, t): b0 = B(8q + t, 8w + g),
    // b1 = B(8q + t + 4, 8w + g), B(k, n) = Wh[row(n) + k * gw] (n = gate * 16 + jj);
    // loaded coalesced along n and scattered into the fragment layout
    // one float4 fragment {b0_hi, b1_hi, b0_lo, b1_lo} per (k-step, warp,
    // lane): b0 = B(8q + t, 8w + g), b1 = B(8q + t + 4, 8w + g); kBatch
    // fragments (2 loads each) in flight per thread, conflict-free 16 B stores
    constexpr int kBatch = 8;
    const int nfrag = KS * 8 * 32;
    for (int f0 = tid; f0 < nfrag; f0 += kBatch * kRT) {
      float b0[kBatch], b1[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int fi = f0 + u * kRT;
        const int q = fi >> 8, w = (fi >> 5) & 7, l = fi & 31;
        const int n = 8 * w + (l >> 2), k = 8 * q + (l & 3);
        const int gate = n / kU, j = j0 + (n - gate * kU);
        const float* src = C.Wh + goff[gate] + j + (int64_t)k * C.gw;
        const bool ok = fi < nfrag && j < C.H;
        b0[u] = ok && k < C.H ? __ldg(src) : 0.f;
        b1[u] = ok && k + 4 < C.H ? __ldg(src + (int64_t)4 * C.gw) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int fi = f0 + u * kRT;
        if (fi >= nfrag) break;
        Bf[fi] = make_float4(__uint_as_float(tf32_hi(b0[u])), __uint_as_float(tf32_hi(b1[u])),
                             __uint_as_float(tf32_lo(b0[u])), __uint_as_float(tf32_lo(b1[u])));
      }
    }
    if (a.trace == 2 && tid == 0) trace(0, 252);
    if (tid < kRnnSlots) sp[0].p[tid] = C.val[tid];
    if (tid == kRnnSlots) sp[0].b1 = C.b1[0];
    // h buffers: zero (padding columns stay zero), then h_{-1} into buffer 1
    for (int idx = tid; idx < 2 * BS * HP; idx += kRT) hS[idx] = 0.f;
    if (tid == 0) {
      // every (row, unit) of a slice is pushed by its owner once per step
      const uint32_t bytes = (uint32_t)(BS * C.H * 4);
      mbar_init_cl(&h_full[0], 1);
      mbar_init_cl(&h_full[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (C.T > 1) mbar_arm(&h_full[0], bytes);  // h_0
      if (C.T > 2) mbar_arm(&h_full[1], bytes);  // h_1
    }
  }
  // weights and tables above do not depend on the preceding grid (PDL):
  // wait for it only now, so this staging overlaps its tail
  pdl_prologue();
  __syncthreads();
  if (a.trace == 2 && tid == 0) trace(0, 253);
  if (warp < 8) {
    const int fl = fl_hp;
    const float* Hp = Hp0;
    if (a.vec) {
      const int w4 = C.H >> 2;
      for (int idx = tid; idx < BS * w4; idx += kRT) {
        const int b = idx / w4, q = idx - (idx / w4) * w4;
        const int row = b0 + b;
        if (row < C.B)
          cp_async16(hS + (size_t)BS * HP + (size_t)b * HP + 4 * q, Hp + ((fl & 2) ? 0 : (int64_t)row * C.H) + 4 * q);
      }
      cp_async_wait_all();
    } else {  // rows not 16 B aligned (H % 4 != 0): element loads
      for (int idx = tid; idx < BS * C.H; idx += kRT) {
        const int b = idx / C.H, k = idx - (idx / C.H) * C.H;
        const int row = b0 + b;
        if (row < C.B) hS[(size_t)BS * HP + (size_t)b * HP + k] = Hp[((fl & 2) ? 0 : (int64_t)row * C.H) + k];
      }
    }
  }
  __syncthreads();
  if (a.trace == 2 && tid == 0) trace(0, 254);
  cluster_sync_all();  // every peer is resident and initialised before any DSMEM push
  if (a.trace && tid == 0) trace(0, 1);
  if (warp == 8) return;  // no cross-chain signalling in gx mode

  const int cb = tid / kU, cj = tid - (tid / kU) * kU;
  const int crow = b0 + cb, cjj = j0 + cj;
  const bool cell_mine = cb < BS && crow < C.B && cjj < C.H;
  const bool cell_row = cb < BS;
  float c_carry = 0.f;
  const uint32_t h_local0 = smem_addr(hS + (size_t)(cb < BS ? cb : 0) * HP + cjj);

  for (int t = 0; t < C.T; ++t) {
    const StepPtrs& P = sp[t & 1];
    const float* nxt = nullptr;
    int nxt_b1 = 0;
    if (warp == 1 && t + 1 < C.T) {
      if (lane < kRnnSlots) nxt = C.val[(size_t)(t + 1) * kRnnSlots + lane];
      if (lane == kRnnSlots) nxt_b1 = C.b1[t + 1];
    }
    const int fl = P.b1;
    if (t == 0 && cell_mine) c_carry = __ldcg(P.p[S_CP] + ((fl & 4) ? cjj : (int64_t)crow * C.H + cjj));
    float gx[4] = {0.f, 0.f, 0.f, 0.f};
    if (cell_mine) {
      const float* Gr = P.p[S_G] + (int64_t)crow * C.gw;
      gx[0] = Gr[C.off_i + cjj];
      gx[1] = Gr[C.off_f + cjj];
      gx[2] = Gr[C.off_o + cjj];
      gx[3] = Gr[C.off_g + cjj];
    }
    if (a.trace == 2 && tid == 0) trace(0, 64 + 4 * t);
    if (t > 0) {
      // h_{t-1}: buffer (t-1)&1, phase (t-1)>>1; then re-arm it for h_{t+1}
      mbar_wait_cl(&h_full[(t - 1) & 1], ((t - 1) >> 1) & 1);
      if (tid == 0 && t + 2 < C.T) mbar_arm(&h_full[(t - 1) & 1], (uint32_t)(BS * C.H * 4));
    }
    if (a.trace == 2 && tid == 0) trace(0, 64 + 4 * t + 1);
    {
      const float* hb = hS + (size_t)((t - 1) & 1) * BS * HP;
      const float* r0 = hb + (size_t)g8 * HP;
      const float* r1 = hb + (size_t)(g8 + 8) * HP;
      const bool v0 = g8 < BS, v1 = g8 + 8 < BS;
      // six independent accumulator chains (3 products x even/odd k-steps)
      float ac[6][4];
#pragma unroll
      for (int z = 0; z < 6; ++z) ac[z][0] = ac[z][1] = ac[z][2] = ac[z][3] = 0.f;
      const float4* bw = Bf + warp * 32 + lane;
#pragma unroll 4
      for (int q = 0; q < KS; ++q) {
        const int k = 8 * q + t4;
        float av[4];
        av[0] = v0 ? r0[k] : 0.f;
        av[1] = v1 ? r1[k] : 0.f;
        av[2] = v0 ? r0[k + 4] : 0.f;
        av[3] = v1 ? r1[k + 4] : 0.f;
        const float4 b = bw[(size_t)q * 256];
        uint32_t ah[4], al[4];
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          ah[z] = step_hi(av[z]);
          al[z] = step_lo(av[z], ah[z]);
        }
        float* c3 = ac[(q & 1) * 3];
        mma_1688(c3, al, __float_as_uint(b.x), __float_as_uint(b.y));
        mma_1688(c3 + 4, ah, __float_as_uint(b.z), __float_as_uint(b.w));
        mma_1688(c3 + 8, ah, __float_as_uint(b.x), __float_as_uint(b.y));
      }
      float acc[4];
#pragma unroll
      for (int z = 0; z < 4; ++z)
        acc[z] = ((ac[0][z] + ac[3][z]) + (ac[1][z] + ac[4][z])) + (ac[2][z] + ac[5][z]);
      // C fragment: rows g8 / g8+8, columns 8w + 2 t4 (+1)
      float* o0 = gS + (size_t)g8 * (kCU + 4) + 8 * warp + 2 * t4;
      if (v0) *reinterpret_cast<float2*>(o0) = make_float2(acc[0], acc[1]);
      if (v1) *reinterpret_cast<float2*>(o0 + 8 * (kCU + 4)) = make_float2(acc[2], acc[3]);
    }
    csync();
    if (a.trace == 2 && tid == 0) trace(0, 64 + 4 * t + 2);
    float x4[4] = {0.f, 0.f, 0.f, 0.f}, ai = 0.f, af = 0.f, ao = 0.f, ag = 0.f, ig = 0.f, p = 0.f, c = 0.f, tc = 0.f;
    float h = 0.f;
    const int64_t r = (int64_t)crow * C.H + cjj;
    if (cell_mine) {
      const float* gr = gS + (size_t)cb * (kCU + 4) + cj;
#pragma unroll
      for (int gate = 0; gate < 4; ++gate) x4[gate] = gx[gate] + gr[gate * kU];
      ai = sigmoid_ref(x4[0]);
      af = sigmoid_ref(x4[1]);
      ao = sigmoid_ref(x4[2]);
      ag = tanhf(x4[3]);
      ig = ai * ag;
      p = af * c_carry;
      c = ig + p;
      c_carry = c;
      tc = tanhf(c);
      h = ao * tc;
    }
    if (a.trace == 2 && tid == 0) trace(0, 64 + 4 * t + 3);
    if (t + 1 < C.T) {
      // push h_t into buffer t&1 of every CTA of the cluster: the 4 units of
      // a quad (consecutive lanes of one row) are gathered into the quad's
      // first lane, one 16 B st.async per peer (a quarter of the DSMEM
      // transactions); a ragged last quad pushes per element
      const float h1 = __shfl_down_sync(0xffffffffu, h, 1);
      const float h2 = __shfl_down_sync(0xffffffffu, h, 2);
      const float h3 = __shfl_down_sync(0xffffffffu, h, 3);
      const bool full_quad = (cjj | 3) < C.H;
      if (cell_row && cjj < C.H && (!full_quad || (cj & 3) == 0)) {
        const uint32_t la = h_local0 + (uint32_t)((t & 1) * BS * HP * 4);
        const uint32_t lb = smem_addr(&h_full[t & 1]);
        if (full_quad) {
          const float4 v = make_float4(h, h1, h2, h3);
          for (int q = 0; q < C.n_u; ++q) st_async_v4(mapa(la, q), v, mapa(lb, q));
        } else {
          for (int q = 0; q < C.n_u; ++q) st_async_f32(mapa(la, q), h, mapa(lb, q));
        }
      }
    }
    if (warp == 1 && t + 1 < C.T) {
      if (lane < kRnnSlots) sp[(t + 1) & 1].p[lane] = nxt;
      if (lane == kRnnSlots) sp[(t + 1) & 1].b1 = nxt_b1;
    }
    csync();  // sp of step t+1 published; gS free for reuse
    if (a.trace && tid == 0) trace(0, 2 + t);
    if (cell_mine) {
      const_cast<float*>(P.p[S_H])[r] = h;
      float* G = const_cast<float*>(P.p[S_G]) + (int64_t)crow * C.gw;
      G[C.off_i + cjj] = x4[0];
      G[C.off_f + cjj] = x4[1];
      G[C.off_o + cjj] = x4[2];
      G[C.off_g + cjj] = x4[3];
      auto W = [&](int slot, float v) { const_cast<float*>(P.p[slot])[r] = v; };
      W(S_PI, x4[0]);
      W(S_PF, x4[1]);
      W(S_PO, x4[2]);
      W(S_PG, x4[3]);
      W(S_AI, ai);
      W(S_AF, af);
      W(S_AO, ao);
      W(S_AG, ag);
      W(S_IG, ig);
      W(S_FC, p);
      W(S_C, c);
      W(S_TC, tc);
    }
  }
}

// Backward recurrence (no stacked consumer: the layer above's dX is a batched
// GEMM): per step the cell backward of this CTA's (16 rows x 16 units), then
// the reduce-scatter dh_{t-1}[rows, all units] = dG_t[rows, own 64 gate cols]
// Wh[own cols, :] on the tensor cores (warp w owns unit tiles 4w..4w+3 of 8,
// 3xTF32 mma.sync, K = 64), each partial pushed to the unit owner's slot with
// st.async (transaction bytes on the owner's mbarrier); the owner sums the n_u
// slots in rank order (deterministic).
template <int BS>
__global__ void __launch_bounds__(kClThreads, 1) rnn_bwd_cl_kernel(const __grid_constant__ RnnArgs a) {
  // (pdl_prologue after the weight staging below)
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ StepPtrs2 sp[2];
  __shared__ __align__(8) uint64_t rec_full[2];
  const int ci = chain_of(a, blockIdx.x);
  const RnnChain C = a.ch[ci];  // register copy (dynamic-index constant loads are slow)
  const int local = blockIdx.x - C.cta0;
  const int s = local / C.n_u, ub = local - (local / C.n_u) * C.n_u;
  const int b0 = s * BS, j0 = ub * kU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int HU = C.n_u * kU;                    // units covered by the cluster (>= H)
  const int NT = HU / 8;                        // unit tiles of 8
  const int goff[4] = {C.off_i, C.off_f, C.off_o, C.off_g};
  float4* Bf = reinterpret_cast<float4*>(sm);   // [NT][8 k-steps][32 lanes] Wh fragments (hi, lo)
  float* dGl = sm + (size_t)NT * 8 * 32 * 4;    // [BS][64 + 4] own gate gradients (A operand)
  float* recv = dGl + (size_t)BS * (kCU + 4);   // [2][n_u][BS][16] reduce-scatter slots
  const uint32_t slot_bytes = (uint32_t)(C.n_u * BS * kU * 4);
  if (a.trace && tid == 0) trace(1, 0);

  if (warp < 8) {
    // B(k, n) = Wh[row(k) + n * gw], k = own gate column (gate * 16 + jj), n = unit;
    // fragment (nt, q, lane = g*4 + t): b0 = B(8q + t, 8nt + g), b1 = B(8q + t + 4, 8nt + g)
    // one float4 fragment per (unit tile, k-step, lane), 2 loads each,
    // kBatch in flight per thread, conflict-free 16 B stores
    constexpr int kBatch = 8;
    const int nfrag = NT * 8 * 32;
    for (int f0 = tid; f0 < nfrag; f0 += kBatch * kRT) {
      float b0[kBatch], b1[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int fi = f0 + u * kRT;
        const int nt = fi >> 8, q = (fi >> 5) & 7, l = fi & 31;
        const int n = 8 * nt + (l >> 2), k = 8 * q + (l & 3);
        const int gate = k / kU, jj = j0 + (k - gate * kU);
        const float* src = C.Wh + goff[gate] + jj + (int64_t)n * C.gw;
        const bool ok = fi < nfrag && n < C.H;
        b0[u] = ok && jj < C.H ? __ldg(src) : 0.f;
        b1[u] = ok && jj + 4 < C.H ? __ldg(src + 4) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int fi = f0 + u * kRT;
        if (fi >= nfrag) break;
        Bf[fi] = make_float4(__uint_as_float(tf32_hi(b0[u])), __uint_as_float(tf32_hi(b1[u])),
                             __uint_as_float(tf32_lo(b0[u])), __uint_as_float(tf32_lo(b1[u])));
      }
    }
    {
      const int t = C.T - 1;
      if (tid < kRnnSlots) sp[t & 1].v[tid] = C.val[(size_t)t * kRnnSlots + tid];
      if (tid >= 32 && tid < 32 + kRnnSlots) sp[t & 1].d[tid - 32] = C.grad[(size_t)t * kRnnSlots + tid - 32];
      if (tid == 64) sp[t & 1].b1 = C.b1[t];
    }
    for (int idx = tid; idx < BS * (kCU + 4); idx += kRT) dGl[idx] = 0.f;
    if (tid == 0) {
      mbar_init_cl(&rec_full[0], 1);
      mbar_init_cl(&rec_full[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const int R = C.T - 1 + (C.h0 ? 1 : 0);  // reduce-scatter rounds (+1: dh_{-1})
      if (R > 0) mbar_arm(&rec_full[0], slot_bytes);  // iteration 0
      if (R > 1) mbar_arm(&rec_full[1], slot_bytes);  // iteration 1
    }
  }
  pdl_prologue();  // weight staging above overlaps the preceding grid
  __syncthreads();
  cluster_sync_all();
  if (a.trace && tid == 0) trace(1, 1);
  if (warp == 8) return;

  const int cb = tid / kU, cj = tid - (tid / kU) * kU;
  const int row = b0 + cb, j = j0 + cj;
  const bool mine = cb < BS && row < C.B && j < C.H;
  const int64_t r = (int64_t)row * C.H + j;
  const uint32_t my_rank = cluster_rank();
  const uint32_t recv_local = smem_addr(recv);
  const uint32_t bar_local = smem_addr(&rec_full[0]);
  const int g8 = lane >> 2, t4 = lane & 3;
  const int R = C.T - 1 + (C.h0 ? 1 : 0);
  float rec = 0.f, dc_carry = 0.f;
  float ao = 0.f, ai = 0.f, ag = 0.f, tc = 0.f, af = 0.f, ck = 0.f, gh_ext = 0.f, gc_ext = 0.f;
  auto load_cell = [&](const StepPtrs2& P) {
    if (!mine) return;
    const bool cb1 = (P.b1 & 4) != 0;
    ao = P.v[S_AO][r];
    ai = P.v[S_AI][r];
    ag = P.v[S_AG][r];
    tc = P.v[S_TC][r];
    af = P.v[S_AF][r];
    ck = P.v[S_CP][cb1 ? j : r];
    gh_ext = P.d[S_H][r];
    gc_ext = P.d[S_C][r];
  };
  load_cell(sp[(C.T - 1) & 1]);

  for (int t = C.T - 1, it = 0; t >= 0; --t, ++it) {
    const StepPtrs2& P = sp[t & 1];
    const float* nv = nullptr;
    float* nd = nullptr;
    int nb1 = 0;
    if (warp == 1 && t > 0) {
      if (lane < kRnnSlots) {
        nv = C.val[(size_t)(t - 1) * kRnnSlots + lane];
        nd = C.grad[(size_t)(t - 1) * kRnnSlots + lane];
      }
      if (lane == kRnnSlots) nb1 = C.b1[t - 1];
    }
    const bool cb1 = (P.b1 & 4) != 0;
    float gh = 0.f, d_tc = 0.f, d_o = 0.f, dc = 0.f, d_i = 0.f, d_g = 0.f, dpi = 0.f, dpo = 0.f, dpg = 0.f;
    float d_f = 0.f, dpf = 0.f;
    if (mine) {
      gh = gh_ext + rec;
      d_tc = gh * ao;
      d_o = gh * tc;
      dc = (gc_ext + dc_carry) + (1.f - tc * tc) * d_tc;
      d_i = dc * ag;
      d_g = dc * ai;
      dpi = ai * (1.f - ai) * d_i;
      dpo = ao * (1.f - ao) * d_o;
      dpg = (1.f - ag * ag) * d_g;
      d_f = dc * ck;
      dpf = af * (1.f - af) * d_f;
      dc_carry = dc * af;
    }
    if (t > 0 || C.h0) {  // t == 0: the round that yields dh_{-1}
      if (cb < BS) {
        float* dl = dGl + (size_t)cb * (kCU + 4);
        dl[0 * kU + cj] = dpi;
        dl[1 * kU + cj] = dpf;
        dl[2 * kU + cj] = dpo;
        dl[3 * kU + cj] = dpg;
      }
      csync();
      {
        const float* r0 = dGl + (size_t)g8 * (kCU + 4);
        const float* r1 = dGl + (size_t)(g8 + 8) * (kCU + 4);
        const bool v0 = g8 < BS, v1 = g8 + 8 < BS;
        uint32_t ah[8][4], al[8][4];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int k = 8 * q + t4;
          const float av[4] = {v0 ? r0[k] : 0.f, v1 ? r1[k] : 0.f, v0 ? r0[k + 4] : 0.f, v1 ? r1[k + 4] : 0.f};
#pragma unroll
          for (int z = 0; z < 4; ++z) {
            ah[q][z] = step_hi(av[z]);
            al[q][z] = step_lo(av[z], ah[q][z]);
          }
        }
        const uint32_t rbase = recv_local + 4u * (uint32_t)(((it & 1) * C.n_u + (int)my_rank) * BS * kU);
        for (int nt = warp; nt < NT; nt += 8) {
          float ac[3][4];
#pragma unroll
          for (int z = 0; z < 3; ++z) ac[z][0] = ac[z][1] = ac[z][2] = ac[z][3] = 0.f;
          const float4* bw = Bf + (size_t)nt * 256 + lane;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b = bw[q * 32];
            mma_1688(ac[0], al[q], __float_as_uint(b.x), __float_as_uint(b.y));
            mma_1688(ac[1], ah[q], __float_as_uint(b.z), __float_as_uint(b.w));
            mma_1688(ac[2], ah[q], __float_as_uint(b.x), __float_as_uint(b.y));
          }
          // C fragment rows g8 / g8+8, units 8nt + 2t4 (+1) -> owner slot [my_rank]
          const int u0 = 8 * nt + 2 * t4;
          const int owner = u0 / kU, uo = u0 - owner * kU;
          const uint32_t rb = mapa(bar_local + 8 * (it & 1), owner);
          if (v0)
            st_async_v2(mapa(rbase + 4u * (uint32_t)(g8 * kU + uo), owner),
                        make_float2(ac[0][0] + ac[1][0] + ac[2][0], ac[0][1] + ac[1][1] + ac[2][1]), rb);
          if (v1)
            st_async_v2(mapa(rbase + 4u * (uint32_t)((g8 + 8) * kU + uo), owner),
                        make_float2(ac[0][2] + ac[1][2] + ac[2][2], ac[0][3] + ac[1][3] + ac[2][3]), rb);
        }
      }
      if (warp == 1 && t > 0) {
        if (lane < kRnnSlots) {
          sp[(t - 1) & 1].v[lane] = nv;
          sp[(t - 1) & 1].d[lane] = nd;
        }
        if (lane == kRnnSlots) sp[(t - 1) & 1].b1 = nb1;
      }
      csync();  // sp of step t-1 published; dGl free for reuse
    }
    if (a.trace && tid == 0) trace(1, 2 + t);
    if (mine) {
      float* const* D = P.d;
      float* dG = D[S_G] + (int64_t)row * C.gw;
      dG[C.off_i + j] = dpi;
      dG[C.off_o + j] = dpo;
      dG[C.off_g + j] = dpg;
      dG[C.off_f + j] = dpf;
      D[S_H][r] = gh;
      D[S_TC][r] = d_tc;
      D[S_AO][r] = d_o;
      D[S_C][r] = dc;
      D[S_IG][r] = dc;
      D[S_AI][r] = d_i;
      D[S_AG][r] = d_g;
      D[S_PI][r] = dpi;
      D[S_PO][r] = dpo;
      D[S_PG][r] = dpg;
      D[S_FC][r] = dc;
      D[S_AF][r] = d_f;
      D[S_PF][r] = dpf;
      if (t == 0 && !cb1) D[S_CP][r] += dc_carry;
    }
    if (t > 0 || C.h0) {
      if (t > 0) load_cell(sp[(t - 1) & 1]);
      mbar_wait_cl(&rec_full[it & 1], (it >> 1) & 1);
      if (tid == 0 && it + 2 <= R - 1) mbar_arm(&rec_full[it & 1], slot_bytes);
      rec = 0.f;
      if (cb < BS) {
        const float* slot = recv + (size_t)(it & 1) * C.n_u * BS * kU + (size_t)cb * kU + cj;
        for (int q = 0; q < C.n_u; ++q) rec += slot[(size_t)q * BS * kU];
      }
    }
  }
  // initial-state gradients (t = -1), replacing a dX GEMM + row reduce and
  // rnn_c0_kernel launch per chain: rec now holds dh_{-1}[row, j], dc_carry
  // the batch-1 c_{-1} term dc_0 * f_0 of (row, j)
  if (C.h0 == 1 && mine) sp[0].d[S_HP][r] += rec;  // per-row h_{-1}
  if (C.h0 == 2 || C.c0) {
    // batch-1 targets: this slice's rows summed in fixed order into
    // part[s][j] (the slices' partials are summed by rnn_part_sum_kernel)
    __shared__ float red[2][16][kU + 1];
    if (cb < BS) {
      red[0][cb][cj] = mine ? rec : 0.f;
      red[1][cb][cj] = mine ? dc_carry : 0.f;
    }
    csync();
    if (tid < 2 * kU) {
      const int which = tid / kU, u = tid - which * kU;
      float* part = which == 0 ? (C.h0 == 2 ? C.h0_part : nullptr) : (C.c0 ? C.c0_part : nullptr);
      if (part && j0 + u < C.H) {
        float acc = 0.f;
        for (int b = 0; b < BS; ++b) acc += red[which][b][u];
        part[(size_t)s * C.H + j0 + u] = acc;
      }
    }
  }
}

// dst[u] += sum_s part[s][u] over the batch slices of each item, items in
// order, one block (initial-state gradients of batch-1 h_{-1} / c_{-1})
__global__ void rnn_part_sum_kernel(RnnPartSum a) {
  pdl_prologue();
  for (int k = 0; k < a.n; ++k) {
    for (int u = threadIdx.x; u < a.H[k]; u += blockDim.x) {
      float acc = 0.f;
      for (int q = 0; q < a.n_s[k]; ++q) acc += a.part[k][(size_t)q * a.H[k] + u];
      a.dst[k][u] += acc;
    }
    __syncthreads();  // a later item may target the same node
  }
}

// dst[u] += sum_b dc0[b][u] * af0[b][u]  (batch-1 c_{-1} of each listed chain)
__global__ void rnn_c0_kernel(RnnC0 a) {
  pdl_prologue();
  // block = (chain k, 32 units); 8 warps split the batch, fixed-order reduce
  __shared__ float red[8][32];
  int k = 0, base = 0;
  const int blk = blockIdx.x;
  while (k < a.n && blk >= base + (a.H[k] + 31) / 32) base += (a.H[k++] + 31) / 32;
  if (k >= a.n) return;
  const int u = (blk - base) * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
  const int H = a.H[k], B = a.B[k];
  float s = 0.f;
  if (u < H)
    for (int b = w; b < B; b += 8) s += a.dc[k][(int64_t)b * H + u] * a.af[k][(int64_t)b * H + u];
  red[w][threadIdx.x & 31] = s;
  __syncthreads();
  if (w == 0 && u < H) {
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][threadIdx.x];
    a.dst[k][u] += t;
  }
}

// per-kernel one-time attribute setup: the dynamic shared memory limit is
// raised to the opt-in maximum once (cudaFuncSetAttribute is not free)
constexpr int kSmemOptin = 227 * 1024;
template <class K>
bool smem_attr_once(K k, bool nonportable_cluster) {
  static std::mutex mu;
  static std::vector<const void*> done;
  std::lock_guard<std::mutex> lk(mu);
  const void* key = reinterpret_cast<const void*>(k);
  for (const void* d : done)
    if (d == key) return true;
  int dev = 0, optin = kSmemOptin;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return false;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes) !=
      cudaSuccess)
    return false;
  if (nonportable_cluster && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return false;
  done.push_back(key);
  return true;
}

template <int BS>
int launch_fwd_bs(const RnnArgs& a, size_t smem, cudaStream_t s) {
  auto k = rnn_fwd_kernel<BS>;
  if (!smem_attr_once(k, false)) return -1;
  void* args[] = {const_cast<RnnArgs*>(&a)};
  if (cudaLaunchCooperativeKernel((const void*)k, dim3(a.ctas), dim3(kRT), args, smem, s) != cudaSuccess) return -1;
  return 1;
}

template <int BS>
int launch_bwd_bs(const RnnArgs& a, size_t smem, cudaStream_t s) {
  auto k = rnn_bwd_kernel<BS>;
  if (!smem_attr_once(k, false)) return -1;
  void* args[] = {const_cast<RnnArgs*>(&a)};
  if (cudaLaunchCooperativeKernel((const void*)k, dim3(a.ctas), dim3(kRT), args, smem, s) != cudaSuccess) return -1;
  return 1;
}

// max co-resident clusters of kernel k at this cluster size and shared
// memory (cached per (kernel, cluster size, 4 KiB smem bucket))
cudaError_t cluster_active(void (*k)(const RnnArgs), const cudaLaunchConfig_t& cfg, int cluster, size_t smem,
                           int* active) {
  static std::mutex mu;
  static std::vector<std::pair<std::tuple<const void*, int, size_t>, int>> memo;
  const auto key = std::make_tuple(reinterpret_cast<const void*>(k), cluster, (smem + 4095) / 4096);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& m : memo)
    if (m.first == key) {
      *active = m.second;
      return cudaSuccess;
    }
  cudaLaunchConfig_t q = cfg;
  q.dynamicSmemBytes = ((smem + 4095) / 4096) * 4096;
  const cudaError_t oe = cudaOccupancyMaxActiveClusters(active, k, &q);
  if (oe == cudaSuccess) memo.push_back({key, *active});
  return oe;
}

template <int BS>
void (*cl_kernel(bool bwd))(const RnnArgs) {
  return bwd ? rnn_bwd_cl_kernel<BS> : rnn_fwd_cl_kernel<BS>;
}

template <int BS>
bool cl_fits_bs(const RnnArgs& a, bool bwd, size_t smem, int cluster) {
  void (*k)(const RnnArgs) = cl_kernel<BS>(bwd);
  if (!smem_attr_once(k, true)) return false;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.ctas);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int active = 0;
  const cudaError_t oe = cluster_active(k, cfg, cluster, smem, &active);
  if (oe != cudaSuccess) cudaGetLastError();
  return oe == cudaSuccess && active * cluster >= a.ctas;
}

template <int BS>
int launch_cl_bs(const RnnArgs& a, bool bwd, size_t smem, int cluster, cudaStream_t s) {
  void (*k)(const RnnArgs) = bwd ? rnn_bwd_cl_kernel<BS> : rnn_fwd_cl_kernel<BS>;
  if (!smem_attr_once(k, true)) return -1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.ctas);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // every cluster must be resident at once (stacked chains wait on each other)
  int active = 0;
  const cudaError_t oe = cluster_active(k, cfg, cluster, smem, &active);
  if (rnn_trace_enabled())
    fprintf(stderr, "[rnn] %s cluster %d smem %zu ctas %d: max active clusters %d (%s)\n", bwd ? "bwd" : "fwd",
            cluster, smem, a.ctas, active, cudaGetErrorString(oe));
  if (oe != cudaSuccess || active * cluster < a.ctas) {
    cudaGetLastError();
    return -2;
  }
  cudaLaunchAttribute at2[2] = {at[0], {}};
  at2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at2[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at2;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, k, a) != cudaSuccess) return -1;
  return 1;
}

}  // namespace

size_t rnn_fwd_cl_smem(int K_in, int H, int bs) {
  (void)K_in;  // gx mode: recurrent input only
  const int KS = (H + 7) / 8;
  return 4 * ((size_t)KS * 8 * 32 * 4 + 2 * (size_t)bs * (8 * KS + 4) + (size_t)bs * (kCU + 4));
}

size_t rnn_bwd_cl_smem(int H, int gw_c, int bs, int cj) {
  (void)gw_c;  // no stacked consumer in the cluster kernel
  (void)cj;
  const int HU = (H + kU - 1) / kU * kU;
  const int nu = HU / kU;
  return 4 * ((size_t)(HU / 8) * 8 * 32 * 4 + (size_t)bs * (kCU + 4) + 2 * (size_t)nu * bs * kU);
}

int rnn_rows_per_cta(int B) { return B >= 16 ? 16 : B >= 8 ? 8 : B >= 4 ? 4 : B >= 2 ? 2 : 1; }

size_t rnn_fwd_smem(int K, int bs) {
  return 4 * ((size_t)K * kCU + (size_t)(K + 4) * bs + 8 * (size_t)bs * kCU + kCU);
}

size_t rnn_bwd_smem(int gw, int gw_c, int bs, int cj) {
  return 4 * ((size_t)gw * kU + (size_t)gw_c * kU + (size_t)(cj + 4) * bs + 8 * (size_t)bs * kU);
}

bool rnn_cluster_enabled() {
  const char* e = std::getenv("DG_RNN_CLUSTER");
  return !(e && e[0] == '0');
}

bool rnn_enabled() {
  const char* e = std::getenv("DG_RNN");
  return !(e && e[0] == '0');
}

bool rnn_cluster_fits(const RnnArgs& a, bool backward, size_t smem, int cluster) {
  switch (a.bs) {
    case 16: return cl_fits_bs<16>(a, backward, smem, cluster);
    case 8: return cl_fits_bs<8>(a, backward, smem, cluster);
    case 4: return cl_fits_bs<4>(a, backward, smem, cluster);
    case 2: return cl_fits_bs<2>(a, backward, smem, cluster);
    default: return cl_fits_bs<1>(a, backward, smem, cluster);
  }
}

int launch_rnn_cluster(const RnnArgs& a, bool backward, size_t smem, int cluster, cudaStream_t s) {
  // global arrival counters only carry cross-chain (stacked) dependencies here
  bool cross = false;
  for (int k = 0; k < a.n_chains; ++k) cross = cross || a.ch[k].src >= 0 || a.ch[k].cons >= 0;
  if (cross && cudaMemsetAsync(a.flags, 0, (size_t)a.n_flags * sizeof(int), s) != cudaSuccess) return -1;
  switch (a.bs) {
    case 16: return launch_cl_bs<16>(a, backward, smem, cluster, s);
    case 8: return launch_cl_bs<8>(a, backward, smem, cluster, s);
    case 4: return launch_cl_bs<4>(a, backward, smem, cluster, s);
    case 2: return launch_cl_bs<2>(a, backward, smem, cluster, s);
    default: return launch_cl_bs<1>(a, backward, smem, cluster, s);
  }
}

int launch_rnn(const RnnArgs& a, bool backward, size_t smem, cudaStream_t s) {
  if (cudaMemsetAsync(a.flags, 0, (size_t)a.n_flags * sizeof(int), s) != cudaSuccess) return -1;
  int n = -1;
  switch (a.bs) {
    case 16: n = backward ? launch_bwd_bs<16>(a, smem, s) : launch_fwd_bs<16>(a, smem, s); break;
    case 8: n = backward ? launch_bwd_bs<8>(a, smem, s) : launch_fwd_bs<8>(a, smem, s); break;
    case 4: n = backward ? launch_bwd_bs<4>(a, smem, s) : launch_fwd_bs<4>(a, smem, s); break;
    case 2: n = backward ? launch_bwd_bs<2>(a, smem, s) : launch_fwd_bs<2>(a, smem, s); break;
    default: n = backward ? launch_bwd_bs<1>(a, smem, s) : launch_fwd_bs<1>(a, smem, s); break;
  }
  return n;
}

int rnn_trace_read(unsigned long long* host, size_t n) {
  const size_t bytes = sizeof(unsigned long long) * 2 * kSmCountTrace * kTraceSlots;
  if (n * sizeof(unsigned long long) < bytes) return -1;
  return cudaMemcpyFromSymbol(host, g_rnn_trace, bytes) == cudaSuccess ? 0 : -1;
}

bool rnn_trace_enabled() {
  const char* e = std::getenv("DG_RNN_TRACE");
  return e && (e[0] == '1' || e[0] == '2');
}

int launch_rnn_part_sum(const RnnPartSum& a, cudaStream_t s) {
  if (a.n == 0) return 0;
  launch_k(rnn_part_sum_kernel, 1, 256, 0, s, a);
  return 1;
}

int launch_rnn_c0(const RnnC0& a, cudaStream_t s) {
  int blocks = 0;
  for (int k = 0; k < a.n; ++k) blocks += (a.H[k] + 31) / 32;
  if (blocks == 0) return 0;
  launch_k(rnn_c0_kernel, blocks, 256, 0, s, a);
  return 1;
}

}  // namespace dg
