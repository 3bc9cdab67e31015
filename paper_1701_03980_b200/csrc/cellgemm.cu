// Fused gate affine + gated cell for small batched levels (sm_100a, fp32).
//
// A Tree-LSTM level (builders.py:250-274: gates = affine(b, U1, h1, U2, h2),
// then i, f1, f2, o, g picks and activations, c = i*g + f1*c1 + f2*c2,
// h = o*tanh(c); leaves: gates = affine(b, Wx, x), c = i*g) is two node
// groups in the reference interpreter and two launches in the generic
// executor (a grouped GEMM, then cell_fwd_kernel).  Both are tiny -- a
// handful of rows against a 5H x (2H) weight -- so the launch and the
// dependent memory round trips dominate, and the level loop of a tree makes
// them sequential.  Here one launch does both: CTA c owns hidden units
// [8c, 8c+8), computes every gate row of those units (all gw / H gate blocks,
// so the gate node's value is complete) for every row of the level from
// shared-memory copies of the inputs and its weight slice, then runs the cell
// for its units.  Every node of the pattern keeps its own value slot.
//
// Arithmetic: fp32 FMA, each term's dot product in k order, then
// ((b + W1 x1) + W2 x2) like the reference's affine (ops.py:323-340).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace cgrp = cooperative_groups;

namespace dg {
namespace {

__device__ __forceinline__ float sigmoid_ref(float x) {
  x = fminf(fmaxf(x, -60.f), 60.f);  // ops.py:78-83
  return 1.f / (1.f + expf(-x));
}

// weight rows of this CTA's units (gate row q = blk * kAffCellUnits + uu
// <-> G row blk * H + u0 + uu), kB independent loads in flight per thread (a
// load-store pair per iteration would serialise on latency)
__device__ void stage_weights(const AffCellArgs& a, float* ws, int u0, int U) {
  const CellArgs& c = a.cell;
  const int NR = (c.gw / c.H) * kAffCellUnits;
  const int KP = a.kpad;
  constexpr int kB = 8;
  for (int t = 0; t < a.terms; ++t) {
    const int K = a.K[t], ko = a.koff[t];
    const int kend = (t + 1 < a.terms) ? a.koff[t + 1] : KP;
    const int KT = kend - ko;  // padded width of this term
    const float* W = a.W[t];
    const int totw = KT * NR;  // consecutive threads: consecutive units of one gate block
    for (int i0 = threadIdx.x; i0 < totw; i0 += kB * blockDim.x) {
      float v[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int idx = i0 + i * blockDim.x;
        const int k = idx / NR, q = idx - (idx / NR) * NR;
        const int blk = q / kAffCellUnits, uu = q - blk * kAffCellUnits;
        v[i] = (idx < totw && k < K && uu < U) ? __ldg(W + blk * c.H + u0 + uu + (int64_t)k * c.gw) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int idx = i0 + i * blockDim.x;
        if (idx < totw) {
          const int k = idx / NR, q = idx - (idx / NR) * NR;
          ws[(size_t)q * KP + ko + k] = v[i];
        }
      }
    }
  }
}

// one level once the weight rows are in shared memory: inputs, gate rows,
// the gate node's value, the cell (same arithmetic as cell_fwd_kernel)
__device__ void level_fwd(const AffCellArgs& a, const float* ws, float* xs, float* gs, float** sval,
                          const float* (*xrow)[64], int u0, int U) {
  const CellArgs& c = a.cell;
  const int NR = (c.gw / c.H) * kAffCellUnits;
  const int KP = a.kpad;
  const int R = a.rows;
  constexpr int kB = 8;
  // slot pointers of every cell and the input row pointers: one global load
  // each instead of one per element use
  for (int i = threadIdx.x; i < c.nslot * c.n; i += blockDim.x) sval[i] = const_cast<float*>(c.val[i]);
  for (int i = threadIdx.x; i < a.terms * R; i += blockDim.x) xrow[i / R][i % R] = a.x[i / R][i % R];
  __syncthreads();
  for (int t = 0; t < a.terms; ++t) {
    const int K = a.K[t], ko = a.koff[t];
    const int kend = (t + 1 < a.terms) ? a.koff[t + 1] : KP;
    const int KT = kend - ko;
    const int totx = R * KT;
    for (int i0 = threadIdx.x; i0 < totx; i0 += kB * blockDim.x) {
      float v[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int idx = i0 + i * blockDim.x;
        const int r = idx / KT, k = idx - (idx / KT) * KT;
        v[i] = (idx < totx && k < K) ? xrow[t][r][k] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int idx = i0 + i * blockDim.x;
        if (idx < totx) xs[(size_t)(idx / KT) * KP + ko + idx % KT] = v[i];
      }
    }
  }
  __syncthreads();
  // gate rows: every (row, gate row) dot split into L k-parts (one thread
  // each, 4-aligned chunks in k order), the parts summed in order after
  const int pairs = R * NR;
  int L = 1;
  while (L < 8 && pairs * L * 2 <= (int)blockDim.x) L *= 2;
  float* part = gs + (size_t)R * NR;  // [L][pairs] per term (terms summed in order below)
  for (int t = 0; t < a.terms; ++t) {
    const int n4 = (a.K[t] + 3) >> 2;
    const int c4 = (n4 + L - 1) / L;
    for (int p = threadIdx.x; p < pairs * L; p += blockDim.x) {
      const int l = p / pairs, pr = p - l * pairs;
      const int r = pr / NR, q = pr - r * NR;
      const float4* xr = reinterpret_cast<const float4*>(xs + (size_t)r * KP + a.koff[t]);
      const float4* wr = reinterpret_cast<const float4*>(ws + (size_t)q * KP + a.koff[t]);
      float acc = 0.f;
      const int e = min(n4, (l + 1) * c4);
      for (int k4 = l * c4; k4 < e; ++k4) {
        const float4 x = xr[k4], w = wr[k4];
        acc = fmaf(w.x, x.x, acc);
        acc = fmaf(w.y, x.y, acc);
        acc = fmaf(w.z, x.z, acc);
        acc = fmaf(w.w, x.w, acc);
      }
      part[((size_t)t * L + l) * pairs + pr] = acc;
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < pairs; p += blockDim.x) {
    const int r = p / NR, q = p - r * NR;
    const int blk = q / kAffCellUnits, uu = q - blk * kAffCellUnits;
    if (uu >= U) continue;
    const int grow = blk * c.H + u0 + uu;
    float v = a.bias ? a.bias[grow] : 0.f;
    for (int t = 0; t < a.terms; ++t) {
      float dot = 0.f;
      for (int l = 0; l < L; ++l) dot += part[((size_t)t * L + l) * pairs + p];
      v += dot;
    }
    gs[p] = v;
    const int j = r / c.batch, b = r - j * c.batch;
    sval[j][(int64_t)b * c.gw + grow] = v;  // the gate (affine / matmul) node's value
    if (a.act) sval[c.n + j][(int64_t)b * c.gw + grow] = a.act == 1 ? tanhf(v) : sigmoid_ref(v);
  }
  if (a.cat && blockIdx.x == 0) {  // the concatenate node's value: the staged inputs side by side
    for (int idx = threadIdx.x; idx < R * a.kpad; idx += blockDim.x) {
      const int r = idx / a.kpad, k = idx - (idx / a.kpad) * a.kpad;
      int t = 0, base = 0;
      while (t + 1 < a.terms && k >= a.koff[t + 1]) {
        base += a.K[t];
        ++t;
      }
      const int kk = k - a.koff[t];
      if (kk < a.K[t]) a.cat[r][base + kk] = xs[(size_t)r * a.kpad + k];
    }
  }
  __syncthreads();
  if (a.act) {
    __syncthreads();
    return;
  }
  const int m = c.m;
  const int s_pick0 = 1 + m, s_act0 = s_pick0 + 3 + m, s_prod0 = s_act0 + 3 + m, s_add0 = s_prod0 + 1 + m;
  const int s_tc = s_add0 + m, s_h = s_tc + 1;
  const int bi = c.off_i / c.H, bo = c.off_o / c.H, bg = c.off_g / c.H;
  for (int p = threadIdx.x; p < R * U; p += blockDim.x) {
    const int r = p / U, uu = p - r * U;
    const int j = r / c.batch, b = r - j * c.batch;
    const int u = u0 + uu;
    const int64_t rr = (int64_t)b * c.H + u;
    auto V = [&](int slot) { return sval[slot * c.n + j]; };
    const float* gr = gs + (size_t)r * NR + uu;
    const float xi = gr[bi * kAffCellUnits], xo = gr[bo * kAffCellUnits], xg = gr[bg * kAffCellUnits];
    float xf[2] = {0.f, 0.f}, ck[2] = {0.f, 0.f};
    for (int k = 0; k < m; ++k) {
      xf[k] = gr[(c.off_f[k] / c.H) * kAffCellUnits];
      ck[k] = V(1 + k)[rr];
    }
    V(s_pick0)[rr] = xi;
    V(s_pick0 + 1 + m)[rr] = xo;
    V(s_pick0 + 2 + m)[rr] = xg;
    const float ai = sigmoid_ref(xi), ao = sigmoid_ref(xo), ag = tanhf(xg);
    V(s_act0)[rr] = ai;
    V(s_act0 + 1 + m)[rr] = ao;
    V(s_act0 + 2 + m)[rr] = ag;
    float cv = ai * ag;
    V(s_prod0)[rr] = cv;
    for (int k = 0; k < m; ++k) {
      V(s_pick0 + 1 + k)[rr] = xf[k];
      const float af = sigmoid_ref(xf[k]);
      V(s_act0 + 1 + k)[rr] = af;
      const float pk = af * ck[k];
      V(s_prod0 + 1 + k)[rr] = pk;
      cv = cv + pk;
      V(s_add0 + k)[rr] = cv;
    }
    const float tc = tanhf(cv);
    V(s_tc)[rr] = tc;
    V(s_h)[rr] = ao * tc;
  }
  __syncthreads();  // shared buffers are reused by the next level
}

__global__ void __launch_bounds__(256) affine_cell_fwd_kernel(const __grid_constant__ AffCellArgs a) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  const CellArgs& c = a.cell;
  const int u0 = blockIdx.x * kAffCellUnits;
  const int U = min(kAffCellUnits, c.H - u0);
  const int NR = (c.gw / c.H) * kAffCellUnits;
  float* ws = sm;                                   // [NR][KP] weight rows of this CTA's units
  float* xs = ws + (size_t)NR * a.kpad;             // [R][KP] inputs, terms at koff[t] (zero padded)
  float* gs = xs + (size_t)a.rows * a.kpad;         // [R][NR] gate values, then k-part partials
  __shared__ float* sval[20 * 64];
  __shared__ const float* xrow[kAffCellMaxTerms][64];
  stage_weights(a, ws, u0, U);
  pdl_prologue();  // weights above do not depend on the preceding kernel: their loads overlap its tail
  level_fwd(a, ws, xs, gs, sval, xrow, u0, U);
}

// Every level of a tree in ONE launch (Tree-LSTM leaves + compose levels,
// builders.py:250-274): the weight rows of this CTA's units for each weight
// set (leaf Wx, compose U1|U2) are staged once and stay in shared memory for
// every level; a grid-wide barrier separates the levels (a level's inputs
// are the previous levels' h).  Cooperative launch: all CTAs co-resident.
__global__ void __launch_bounds__(256) tree_fwd_kernel(const __grid_constant__ TreeFwdArgs t) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ float* sval[20 * 64];
  __shared__ const float* xrow[kAffCellMaxTerms][64];
  __shared__ AffCellArgs lv;
  const int H = t.H;
  const int u0 = blockIdx.x * kAffCellUnits;
  const int U = min(kAffCellUnits, H - u0);
  float* ws[2] = {sm, sm + t.wfloats[0]};
  float* xs = sm + t.wfloats[0] + t.wfloats[1];
  for (int w = 0; w < t.n_wsets; ++w) stage_weights(t.wset[w], ws[w], u0, U);
  pdl_prologue();
  cgrp::grid_group grid = cgrp::this_grid();
  for (int l = 0; l < t.n_levels; ++l) {
    if (threadIdx.x == 0) lv = t.levels[l];
    __syncthreads();
    const int w = lv.wslot;
    float* gs = xs + (size_t)lv.rows * lv.kpad;
    level_fwd(lv, ws[w], xs, gs, sval, xrow, u0, U);
    if (l + 1 < t.n_levels) {
      __threadfence();
      grid.sync();
    }
  }
}

// Input gradients of a small affine group, dX_t += W_t^T dG (the tree
// levels' gate affines, the tagger's per-word layers): CTA c owns
// kAffCellCols input columns (of the terms' concatenation); it stages the
// rows of W_t^T for them before waiting on the preceding kernel (weights do
// not change during backward), then reads the group's dG rows once and adds
// its columns of dX into the input rows' gradient slots.  The generic path
// is the grouped split-K GEMM, whose dependent loads dominate at a few rows.
// Weight and bias gradients stay in the executor's aggregated dW GEMM /
// column sums.
__global__ void __launch_bounds__(256) affine_dx_small_kernel(const __grid_constant__ AffCellArgs a) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  const int R = a.rows, GW = a.cell.gw;
  int Ktot = 0;
  for (int t = 0; t < a.terms; ++t) Ktot += a.K[t];
  const int kc0 = blockIdx.x * kAffCellCols;
  const int KC = min(kAffCellCols, Ktot - kc0);
  float* wt = sm;                              // [kAffCellCols][GW] rows of W^T (own columns)
  float* dg = wt + (size_t)kAffCellCols * GW;  // [R][GW] gate gradients
  float* part = dg + (size_t)R * GW;           // [L][R * kAffCellCols]
  __shared__ int col_t[kAffCellCols], col_k[kAffCellCols];
  __shared__ float* sgx[kAffCellMaxTerms][64];
  __shared__ const float* sgr[64];
  if (threadIdx.x < kAffCellCols) {
    int kc = kc0 + threadIdx.x, t = 0;
    while (t + 1 < a.terms && kc >= a.K[t]) kc -= a.K[t++];
    col_t[threadIdx.x] = t;
    col_k[threadIdx.x] = kc;
  }
  for (int i = threadIdx.x; i < a.terms * R; i += blockDim.x) sgx[i / R][i % R] = a.gx[i / R][i % R];
  for (int i = threadIdx.x; i < R; i += blockDim.x) sgr[i] = a.grow[i];
  __syncthreads();
  // W_t[:, k] is contiguous (column-major): coalesced, kB loads in flight per
  // thread, before the wait
  constexpr int kB = 8;
  for (int i0 = threadIdx.x; i0 < KC * GW; i0 += kB * blockDim.x) {
    float v[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int idx = i0 + i * blockDim.x;
      const int q = idx / GW, g = idx - (idx / GW) * GW;
      v[i] = idx < KC * GW ? __ldg(a.W[col_t[q]] + g + (int64_t)col_k[q] * GW) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int idx = i0 + i * blockDim.x;
      if (idx < KC * GW) wt[idx] = v[i];
    }
  }
  pdl_prologue();
  for (int i0 = threadIdx.x; i0 < R * GW; i0 += kB * blockDim.x) {
    float v[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int idx = i0 + i * blockDim.x;
      v[i] = idx < R * GW ? sgr[idx / GW][idx % GW] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int idx = i0 + i * blockDim.x;
      if (idx < R * GW) dg[idx] = v[i];
    }
  }
  __syncthreads();
  // (row, column) dots over the gate rows in L parts, summed in order
  const int pairs = R * KC;
  int L = 1;
  while (L < 16 && pairs * L * 2 <= (int)blockDim.x) L *= 2;
  const int cg = (GW + L - 1) / L;
  for (int p = threadIdx.x; p < pairs * L; p += blockDim.x) {
    const int l = p / pairs, pr = p - l * pairs;
    const int r = pr / KC, q = pr - r * KC;
    const float* w = wt + (size_t)q * GW;
    const float* d = dg + (size_t)r * GW;
    float acc = 0.f;
    const int e = min(GW, (l + 1) * cg);
    for (int g = l * cg; g < e; ++g) acc = fmaf(w[g], d[g], acc);
    part[(size_t)l * pairs + pr] = acc;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < pairs; p += blockDim.x) {
    const int r = p / KC, q = p - r * KC;
    float v = 0.f;
    for (int l = 0; l < L; ++l) v += part[(size_t)l * pairs + p];
    float* gx = sgx[col_t[q]][r] + col_k[q];
    *gx += v;
  }
}

}  // namespace

size_t affine_dx_small_smem(int rows, int gw) {
  return 4 * ((size_t)kAffCellCols * gw + (size_t)rows * gw + 16 * (size_t)rows * kAffCellCols);
}

int launch_affine_dx_small(const AffCellArgs& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(affine_dx_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int Ktot = 0;
  for (int t = 0; t < a.terms; ++t) Ktot += a.K[t];
  const int grid = (Ktot + kAffCellCols - 1) / kAffCellCols;
  if (launch_k(affine_dx_small_kernel, grid, 256, affine_dx_small_smem(a.rows, a.cell.gw), s, a) != cudaSuccess)
    return -1;
  return 1;
}

// k-part partial sums of level_fwd: L parts with L * pairs <= max(pairs, 256)
static size_t part_floats(int rows, int NR) {
  return (size_t)kAffCellMaxTerms * std::max<size_t>((size_t)rows * NR, 256);
}

size_t affine_cell_smem(int rows, int kpad, int gw, int H) {
  const int NR = (gw / H) * kAffCellUnits;
  // weight rows, inputs, gate values, k-part partial sums
  return 4 * ((size_t)rows * kpad + (size_t)NR * kpad + (size_t)rows * NR + part_floats(rows, NR));
}

size_t tree_fwd_smem(const TreeFwdArgs& t) {
  // weight sets, then the largest level's inputs + gate values + partials
  size_t lvl = 0;
  for (int w = 0; w < t.n_wsets; ++w) {
    const AffCellArgs& a = t.wset[w];
    const int NR = (a.cell.gw / a.cell.H) * kAffCellUnits;
    lvl = std::max(lvl, (size_t)t.max_rows * a.kpad + (size_t)t.max_rows * NR + part_floats(t.max_rows, NR));
  }
  return 4 * ((size_t)t.wfloats[0] + t.wfloats[1] + lvl);
}

int launch_tree_fwd(const TreeFwdArgs& t, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tree_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int grid = (t.H + kAffCellUnits - 1) / kAffCellUnits;
  void* args[] = {const_cast<TreeFwdArgs*>(&t)};
  if (cudaLaunchCooperativeKernel((const void*)tree_fwd_kernel, dim3(grid), dim3(256), args, tree_fwd_smem(t), s) !=
      cudaSuccess)
    return -1;
  return 1;
}

int launch_affine_cell_fwd(const AffCellArgs& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(affine_cell_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int grid = (a.cell.H + kAffCellUnits - 1) / kAffCellUnits;
  const size_t smem = affine_cell_smem(a.rows, a.kpad, a.cell.gw, a.cell.H);
  if (launch_k(affine_cell_fwd_kernel, grid, 256, smem, s, a) != cudaSuccess) return -1;
  return 1;
}

}  // namespace dg
