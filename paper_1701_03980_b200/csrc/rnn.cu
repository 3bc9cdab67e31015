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
#include <cstdlib>

#include "kernels.cuh"

namespace dg {

namespace {

constexpr int kRT = 256;  // threads per CTA
constexpr int kU = kRnnUnits;
constexpr int kCU = 4 * kU;  // gate columns per CTA

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

__device__ __forceinline__ int chain_of(const RnnArgs& a, int cta) {
  int ci = 0;
  while (ci + 1 < a.n_chains && cta >= a.ch[ci + 1].cta0) ++ci;
  return ci;
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
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ StepPtrs sp[2];
  const int ci = chain_of(a, blockIdx.x);
  const RnnChain& C = a.ch[ci];
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
  const int kper = (K + 7) / 8;
  const int kbeg = warp * kper, kend = min(K, kbeg + kper);
  const int cb = tid / kU, cj = tid - (tid / kU) * kU;  // cell thread: (row, unit)
  const int crow = b0 + cb, cjj = j0 + cj;
  const bool cell_mine = cb < BS && crow < C.B && cjj < C.H;
  float c_carry = 0.f;  // c_{t-1} of this thread's (row, unit), produced by itself

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
    if (tid == 0) {
      if (src_flags) wait_count(src_flags + t, src_need);
      if (t > 0) wait_count(my_flags + t - 1, C.n_u);
    }
    __syncthreads();
    {
      // stage [x_t | h_{t-1}] rows of this slice (L2 -> smem, bypassing L1)
      const float* X = P.p[S_X];
      const float* Hp = P.p[S_HP];
      if (a.vec) {
        const int K4 = K >> 2, Kin4 = C.K_in >> 2;
        for (int idx = tid; idx < BS * K4; idx += kRT) {
          const int b = idx / K4, k4 = idx - (idx / K4) * K4;
          const int row = b0 + b;
          float* dst = inS + (size_t)b * KP + 4 * k4;
          if (row < C.B) {
            const float* src = k4 < Kin4 ? X + ((fl & 1) ? 0 : (int64_t)row * C.K_in) + 4 * k4
                                         : Hp + ((fl & 2) ? 0 : (int64_t)row * C.H) + 4 * (k4 - Kin4);
            cp_async16(dst, src);
          } else {
            *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        cp_async_wait_all();
      } else {
        for (int idx0 = tid; idx0 < BS * K; idx0 += 4 * kRT) {
          float v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int idx = idx0 + q * kRT;
            const int b = idx / K, k = idx - (idx / K) * K;
            const int row = b0 + b;
            v[q] = 0.f;
            if (idx < BS * K && row < C.B)
              v[q] = k < C.K_in ? __ldcg(X + ((fl & 1) ? 0 : (int64_t)row * C.K_in) + k)
                                : __ldcg(Hp + ((fl & 2) ? 0 : (int64_t)row * C.H) + (k - C.K_in));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int idx = idx0 + q * kRT;
            if (idx < BS * K) inS[(size_t)(idx / K) * KP + (idx - (idx / K) * K)] = v[q];
          }
        }
      }
    }
    __syncthreads();
    {
      float acc[TB][TC];
#pragma unroll
      for (int i = 0; i < TB; ++i)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[i][c] = 0.f;
#pragma unroll 4
      for (int k = kbeg; k < kend; ++k) {
        float xa[TB], wv[TC];
#pragma unroll
        for (int i = 0; i < TB; ++i) xa[i] = inS[(size_t)(i * LB + lb) * KP + k];
#pragma unroll
        for (int c = 0; c < TC; ++c) wv[c] = Ws[(size_t)k * kCU + lc * TC + c];
#pragma unroll
        for (int i = 0; i < TB; ++i)
#pragma unroll
          for (int c = 0; c < TC; ++c) acc[i][c] = fmaf(xa[i], wv[c], acc[i][c]);
      }
#pragma unroll
      for (int i = 0; i < TB; ++i)
#pragma unroll
        for (int c = 0; c < TC; ++c) part[(warp * BS + i * LB + lb) * kCU + lc * TC + c] = acc[i][c];
    }
    __syncthreads();
    if (cell_mine) {
      float x4[4];
#pragma unroll
      for (int gate = 0; gate < 4; ++gate) {
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) sum += part[(w * BS + cb) * kCU + gate * kU + cj];
        x4[gate] = bias[gate * kU + cj] + sum;
      }
      const int row = crow, j = cjj;
      float* G = const_cast<float*>(P.p[S_G]) + (int64_t)row * C.gw;
      G[C.off_i + j] = x4[0];
      G[C.off_f + j] = x4[1];
      G[C.off_o + j] = x4[2];
      G[C.off_g + j] = x4[3];
      const int64_t r = (int64_t)row * C.H + j;
      auto W = [&](int slot, float v) { const_cast<float*>(P.p[slot])[r] = v; };
      W(S_PI, x4[0]);
      W(S_PF, x4[1]);
      W(S_PO, x4[2]);
      W(S_PG, x4[3]);
      const float ai = sigmoid_ref(x4[0]), af = sigmoid_ref(x4[1]), ao = sigmoid_ref(x4[2]);
      const float ag = tanhf(x4[3]);
      W(S_AI, ai);
      W(S_AF, af);
      W(S_AO, ao);
      W(S_AG, ag);
      float c = ai * ag;
      W(S_IG, c);
      const float p = af * c_carry;
      W(S_FC, p);
      c = c + p;
      W(S_C, c);
      c_carry = c;
      const float tc = tanhf(c);
      W(S_TC, tc);
      W(S_H, ao * tc);
    }
    if (warp == 1 && t + 1 < C.T) {
      if (lane < kRnnSlots) sp[(t + 1) & 1].p[lane] = nxt;
      if (lane == kRnnSlots) sp[(t + 1) & 1].b1 = nxt_b1;
    }
    __syncthreads();
    if (tid == 0) arrive(my_flags + t);
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
    __syncthreads();
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
    __syncthreads();
  }
  if (active) {
#pragma unroll
    for (int i = 0; i < TB; ++i)
#pragma unroll
      for (int c = 0; c < TC; ++c) part[(warp * BS + i * LB + lb) * kU + lc * TC + c] = acc[i][c];
  }
  __syncthreads();
  const int cb = tid / kU, cu = tid - (tid / kU) * kU;
  float sum = 0.f;
  if (cb < BS) {
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += part[(w * BS + cb) * kU + cu];
  }
  __syncthreads();
  return sum;
}

struct StepPtrs2 {
  const float* v[kRnnSlots];
  float* d[kRnnSlots];
  int b1;
};

template <int BS>
__global__ void __launch_bounds__(kRT, 1) rnn_bwd_kernel(const __grid_constant__ RnnArgs a) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ StepPtrs2 sp[2];
  const int ci = chain_of(a, blockIdx.x);
  const RnnChain& C = a.ch[ci];
  const int local = blockIdx.x - C.cta0;
  const int s = local / C.n_u, ub = local - (local / C.n_u) * C.n_u;
  const int b0 = s * BS, j0 = ub * kU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RnnChain* Cc = C.cons >= 0 ? &a.ch[C.cons] : nullptr;
  const int gw_c = Cc ? Cc->gw : 0;
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

  int* my_flags = a.flags + C.flag0 + s * C.T;
  const int* cons_flags = Cc ? a.flags + Cc->flag0 + s * Cc->T : nullptr;
  const int cb = tid / kU, cj = tid - (tid / kU) * kU;
  const int row = b0 + cb, j = j0 + cj;
  const bool mine = cb < BS && row < C.B && j < C.H;
  const int64_t r = (int64_t)row * C.H + j;
  float rec = 0.f;      // dh_t from step t+1 of this chain
  float dc_carry = 0.f;  // dc_t contribution of step t+1 (f_{t+1} * dc_{t+1})

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
    const int fl = P.b1;
    const bool cb1 = (fl & 4) != 0;
    // forward values and external gradient contributions of this cell: all
    // independent of other CTAs, loaded before any wait
    float ao = 0.f, ai = 0.f, ag = 0.f, tc = 0.f, af = 0.f, ck = 0.f, gh_ext = 0.f, gc_ext = 0.f;
    if (mine) {
      ao = P.v[S_AO][r];
      ai = P.v[S_AI][r];
      ag = P.v[S_AG][r];
      tc = P.v[S_TC][r];
      af = P.v[S_AF][r];
      ck = P.v[S_CP][cb1 ? j : r];
      gh_ext = P.d[S_H][r];
      gc_ext = P.d[S_C][r];
    }
    float cons = 0.f;
    if (Cc) {
      if (tid == 0) wait_count(cons_flags + t, Cc->n_u);
      __syncthreads();
      cons = rows_times_wt<BS>(Cc->grad[(size_t)t * kRnnSlots + S_G], gw_c, C.B, b0, WcT, dGs, a.cj, part,
                               a.vec);
    }
    if (mine) {
      // internal slots have this cell as their only consumer: written, not
      // accumulated; h and c slots add the contributions gathered above
      float* const* D = P.d;
      const float gh = gh_ext + rec + cons;
      D[S_H][r] = gh;
      const float d_tc = gh * ao;
      const float d_o = gh * tc;
      D[S_TC][r] = d_tc;
      D[S_AO][r] = d_o;
      const float dc = (gc_ext + dc_carry) + (1.f - tc * tc) * d_tc;
      D[S_C][r] = dc;
      D[S_IG][r] = dc;
      const float d_i = dc * ag, d_g = dc * ai;
      D[S_AI][r] = d_i;
      D[S_AG][r] = d_g;
      const float dpi = ai * (1.f - ai) * d_i;
      const float dpo = ao * (1.f - ao) * d_o;
      const float dpg = (1.f - ag * ag) * d_g;
      D[S_PI][r] = dpi;
      D[S_PO][r] = dpo;
      D[S_PG][r] = dpg;
      float* dG = D[S_G] + (int64_t)row * C.gw;
      dG[C.off_i + j] = dpi;
      dG[C.off_o + j] = dpo;
      dG[C.off_g + j] = dpg;
      D[S_FC][r] = dc;
      const float d_f = dc * ck;
      D[S_AF][r] = d_f;
      const float dpf = af * (1.f - af) * d_f;
      D[S_PF][r] = dpf;
      dG[C.off_f + j] = dpf;
      dc_carry = dc * af;
      // c_{-1}: external state (batch-1 broadcast: rnn_c0_kernel sums it)
      if (t == 0 && !cb1) D[S_CP][r] += dc_carry;
    }
    if (warp == 1 && t > 0) {
      if (lane < kRnnSlots) {
        sp[(t - 1) & 1].v[lane] = nv;
        sp[(t - 1) & 1].d[lane] = nd;
      }
      if (lane == kRnnSlots) sp[(t - 1) & 1].b1 = nb1;
    }
    __syncthreads();
    if (tid == 0) arrive(my_flags + t);
    if (t > 0) {
      if (tid == 0) wait_count(my_flags + t, C.n_u);
      __syncthreads();
      rec = rows_times_wt<BS>(P.d[S_G], C.gw, C.B, b0, WhT, dGs, a.cj, part, a.vec);
    }
  }
}

// dst[u] += sum_b dc0[b][u] * af0[b][u]  (batch-1 c_{-1} of each listed chain)
__global__ void rnn_c0_kernel(RnnC0 a) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  int k = 0, base = 0;
  while (k < a.n && q >= base + a.H[k]) base += a.H[k++];
  if (k >= a.n) return;
  const int u = q - base;
  float s = 0.f;
  for (int b = 0; b < a.B[k]; ++b) s += a.dc[k][(int64_t)b * a.H[k] + u] * a.af[k][(int64_t)b * a.H[k] + u];
  a.dst[k][u] += s;
}

template <int BS>
int launch_fwd_bs(const RnnArgs& a, size_t smem, cudaStream_t s) {
  auto k = rnn_fwd_kernel<BS>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  void* args[] = {const_cast<RnnArgs*>(&a)};
  if (cudaLaunchCooperativeKernel((const void*)k, dim3(a.ctas), dim3(kRT), args, smem, s) != cudaSuccess) return -1;
  return 1;
}

template <int BS>
int launch_bwd_bs(const RnnArgs& a, size_t smem, cudaStream_t s) {
  auto k = rnn_bwd_kernel<BS>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  void* args[] = {const_cast<RnnArgs*>(&a)};
  if (cudaLaunchCooperativeKernel((const void*)k, dim3(a.ctas), dim3(kRT), args, smem, s) != cudaSuccess) return -1;
  return 1;
}

}  // namespace

int rnn_rows_per_cta(int B) { return B >= 16 ? 16 : B >= 8 ? 8 : B >= 4 ? 4 : B >= 2 ? 2 : 1; }

size_t rnn_fwd_smem(int K, int bs) {
  return 4 * ((size_t)K * kCU + (size_t)(K + 4) * bs + 8 * (size_t)bs * kCU + kCU);
}

size_t rnn_bwd_smem(int gw, int gw_c, int bs, int cj) {
  return 4 * ((size_t)gw * kU + (size_t)gw_c * kU + (size_t)(cj + 4) * bs + 8 * (size_t)bs * kU);
}

bool rnn_enabled() {
  const char* e = std::getenv("DG_RNN");
  return !(e && e[0] == '0');
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

int launch_rnn_c0(const RnnC0& a, cudaStream_t s) {
  int total = 0;
  for (int k = 0; k < a.n; ++k) total += a.H[k];
  if (total == 0) return 0;
  rnn_c0_kernel<<<(total + 255) / 256, 256, 0, s>>>(a);
  return 1;
}

}  // namespace dg
