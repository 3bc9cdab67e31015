// Group kernels of the executor: elementwise, structural, row-wise (softmax /
// pickneglogsoftmax), embedding gather + sorted segmented scatter-add, generic
// matmul/affine fallbacks, and the trainer rules.  sm_100a, fp32.
//
// Semantics restate pkg/src/dyncore/ops.py (forward overwrites, backward
// accumulates into zero-initialised slots) and trainers.py:63-83.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace dg {

namespace {
thread_local bool g_pdl_skip = false;
}
void pdl_skip_next() { g_pdl_skip = true; }
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DG_PDL");
    return !(e && e[0] == '0');
  }();
  if (g_pdl_skip) {
    g_pdl_skip = false;
    return false;
  }
  return on;
}


namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float sigmoidf_ref(float x) {
  // ops.py:78-83: clip to +-60 before exp
  x = fminf(fmaxf(x, -60.f), 60.f);
  return 1.f / (1.f + expf(-x));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------------------ elementwise

__global__ void ew_fwd_kernel(EwArgs a) {
  pdl_prologue();
  const int64_t size = static_cast<int64_t>(a.elem) * a.batch;
  const int64_t total = size * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / size);
    const int64_t r = t - (int64_t)j * size;
    const int64_t e = r % a.elem;
    const float x = a.a[j][a.a_b1 ? e : r];
    float y;
    switch (a.kind) {
      case EW_TANH: y = tanhf(x); break;
      case EW_LOGISTIC: y = sigmoidf_ref(x); break;
      case EW_SCALE: y = x * a.scalar; break;
      case EW_ADD: y = x + a.b[j][a.b_b1 ? e : r]; break;
      default: y = x * a.b[j][a.b_b1 ? e : r]; break;
    }
    a.out[j][r] = y;
  }
}

// no-broadcast backward: one thread per output element
__global__ void ew_bwd_flat_kernel(EwArgs a) {
  pdl_prologue();
  const int64_t size = static_cast<int64_t>(a.elem) * a.batch;
  const int64_t total = size * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / size);
    const int64_t r = t - (int64_t)j * size;
    const float g = a.gout[j][r];
    switch (a.kind) {
      case EW_TANH: {
        const float y = a.oval[j][r];
        a.ga[j][r] += (1.f - y * y) * g;
        break;
      }
      case EW_LOGISTIC: {
        const float y = a.oval[j][r];
        a.ga[j][r] += y * (1.f - y) * g;
        break;
      }
      case EW_SCALE: a.ga[j][r] += a.scalar * g; break;
      default: {
        // both old gradient values are read before either store (a store
        // would otherwise order the second read behind it); x op x keeps
        // the sequential (ga + ca) + cb
        const bool add = a.kind == EW_ADD;
        const float av = add ? 0.f : a.a[j][r], bv = add ? 0.f : a.b[j][r];
        const float ca = add ? g : g * bv, cb = add ? g : g * av;
        float* pa = a.ga[j] + r;
        float* pb = a.gb[j] + r;
        const float oa = *pa, ob = *pb;
        if (pa == pb) {
          *pa = (oa + ca) + cb;
        } else {
          *pa = oa + ca;
          *pb = ob + cb;
        }
        break;
      }
    }
  }
}

// broadcast backward (binary ops): one thread per (node, element) loops over
// the batch so batch-1 operands receive the batch sum (ops.py:69-75)
__global__ void ew_bwd_bcast_kernel(EwArgs a) {
  pdl_prologue();
  const int64_t total = static_cast<int64_t>(a.elem) * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / a.elem);
    const int e = static_cast<int>(t - (int64_t)j * a.elem);
    float acc_a = 0.f, acc_b = 0.f;
    for (int b = 0; b < a.batch; ++b) {
      const int64_t r = (int64_t)b * a.elem + e;
      const float g = a.gout[j][r];
      float ca, cb = 0.f;
      if (a.kind == EW_SCALE) {
        ca = a.scalar * g;
      } else if (a.kind == EW_ADD) {
        ca = g;
        cb = g;
      } else {
        ca = g * a.b[j][a.b_b1 ? e : r];
        cb = g * a.a[j][a.a_b1 ? e : r];
      }
      if (a.a_b1) acc_a += ca; else a.ga[j][r] += ca;
      if (a.kind != EW_SCALE) {
        if (a.b_b1) acc_b += cb; else a.gb[j][r] += cb;
      }
    }
    if (a.a_b1) a.ga[j][e] += acc_a;
    if (a.b_b1 && a.kind != EW_SCALE) a.gb[j][e] += acc_b;
  }
}

__global__ void chain_fwd_kernel(ChainArgs a) {
  pdl_prologue();
  const int64_t total = (int64_t)a.size * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / a.size);
    const int64_t e = t - (int64_t)j * a.size;
    float s = a.ins[j][e] + a.ins[a.n + j][e];
    a.outs[j][e] = s;
    for (int i = 2; i <= a.len; ++i) {
      s = s + a.ins[(int64_t)i * a.n + j][e];
      a.outs[(int64_t)(i - 1) * a.n + j][e] = s;
    }
  }
}

__global__ void chain_bwd_kernel(ChainArgs a) {
  pdl_prologue();
  const int64_t total = (int64_t)a.size * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / a.size);
    const int64_t e = t - (int64_t)j * a.size;
    const float g = a.gfinal[j][e];
    for (int i = 0; i + 1 < a.len; ++i) a.gouts[(int64_t)i * a.n + j][e] += g;
    for (int i = 0; i <= a.len; ++i) a.gins[(int64_t)i * a.n + j][e] += g;
  }
}

// Few long chains (the scalar loss chain): one block per (chain, element)
// prefetches the terms into shared memory, one thread adds them in the same
// left-to-right order, and the block writes the prefixes back in parallel.
__global__ void chain_fwd_seq_kernel(ChainArgs a) {
  pdl_prologue();
  __shared__ float t[1024];
  const int j = blockIdx.x / a.size;
  const int64_t e = blockIdx.x - (int64_t)j * a.size;
  float s = 0.f;
  for (int base = 0; base <= a.len; base += 1024) {
    const int cnt = min(1024, a.len + 1 - base);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) t[i] = a.ins[(int64_t)(base + i) * a.n + j][e];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < cnt; ++i) {
        s = base + i == 0 ? t[i] : s + t[i];
        t[i] = s;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x)
      if (base + i >= 1) a.outs[(int64_t)(base + i - 1) * a.n + j][e] = t[i];
    __syncthreads();
  }
}

// every (slot, element) of a chain whose gradient slots are all distinct
// (checked on the host): g of the last add is added to each independently
// one thread per (target slot, chain, element): the len - 1 intermediate adds
// and the len + 1 inputs each get the final add's gradient.  The final add's
// own slot is the source and is never written (it would race with the reads
// and leave d(final) doubled).
__global__ void chain_bwd_par_kernel(ChainArgs a) {
  pdl_prologue();
  const int64_t per = (int64_t)a.n * a.size;
  const int64_t total = (int64_t)(2 * a.len) * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int slot = static_cast<int>(t / per);
    const int64_t r = t - (int64_t)slot * per;
    const int j = static_cast<int>(r / a.size);
    const int64_t e = r - (int64_t)j * a.size;
    const float g = a.gfinal[j][e];
    if (slot + 1 < a.len) a.gouts[(int64_t)slot * a.n + j][e] += g;
    else a.gins[(int64_t)(slot - (a.len - 1)) * a.n + j][e] += g;
  }
}

// ------------------------------------------------------------ gated cells

struct CellSlots {
  int m, pick0, act0, prod0, add0, tc, h, c;
  __device__ __forceinline__ explicit CellSlots(int m_) : m(m_) {
    pick0 = 1 + m;
    act0 = pick0 + 3 + m;
    prod0 = act0 + 3 + m;
    add0 = prod0 + 1 + m;
    tc = add0 + m;
    h = tc + 1;
    c = m > 0 ? add0 + m - 1 : prod0;
  }
  // gate order inside the pick/act groups: i, f[0..m), o, g
  __device__ __forceinline__ int gi() const { return 0; }
  __device__ __forceinline__ int gf(int k) const { return 1 + k; }
  __device__ __forceinline__ int go() const { return 1 + m; }
  __device__ __forceinline__ int gg() const { return 2 + m; }
};

// One cell per block: the cell's slot pointers are staged in shared memory once.
template <int M>
__global__ void __launch_bounds__(256) cell_fwd_kernel(CellArgs a) {
  pdl_prologue();
  const CellSlots S(M);
  __shared__ const float* sv[20];
  const int64_t per = (int64_t)a.batch * a.H;
  const int bpc = (int)((per + 255) / 256);
  const int j = blockIdx.x / bpc;
  if ((int)threadIdx.x < a.nslot) sv[threadIdx.x] = a.val[(int64_t)threadIdx.x * a.n + j];
  __syncthreads();
  {
    const int64_t r = (int64_t)(blockIdx.x % bpc) * 256 + threadIdx.x;
    if (r >= per) return;
    const int b = static_cast<int>(r / a.H), u = static_cast<int>(r - (int64_t)b * a.H);
    auto V = [&](int slot) { return sv[slot]; };
    const float* G = V(0) + (int64_t)b * a.gw;
    const float xi = G[a.off_i + u], xo = G[a.off_o + u], xg = G[a.off_g + u];
    float xf[M > 0 ? M : 1], ck[M > 0 ? M : 1];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      xf[k] = G[a.off_f[k] + u];
      ck[k] = V(1 + k)[a.cext_b1[k] ? u : r];  // loaded before any store (no store-to-load waits)
    }
    const_cast<float*>(V(S.pick0 + S.gi()))[r] = xi;
    const_cast<float*>(V(S.pick0 + S.go()))[r] = xo;
    const_cast<float*>(V(S.pick0 + S.gg()))[r] = xg;
    const float ai = sigmoidf_ref(xi), ao = sigmoidf_ref(xo), ag = tanhf(xg);
    const_cast<float*>(V(S.act0 + S.gi()))[r] = ai;
    const_cast<float*>(V(S.act0 + S.go()))[r] = ao;
    const_cast<float*>(V(S.act0 + S.gg()))[r] = ag;
    float c = ai * ag;
    const_cast<float*>(V(S.prod0))[r] = c;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const_cast<float*>(V(S.pick0 + S.gf(k)))[r] = xf[k];
      const float af = sigmoidf_ref(xf[k]);
      const_cast<float*>(V(S.act0 + S.gf(k)))[r] = af;
      const float p = af * ck[k];
      const_cast<float*>(V(S.prod0 + 1 + k))[r] = p;
      c = c + p;
      const_cast<float*>(V(S.add0 + k))[r] = c;
    }
    const float tc = tanhf(c);
    const_cast<float*>(V(S.tc))[r] = tc;
    const_cast<float*>(V(S.h))[r] = ao * tc;
  }
}

// kLoopBatch (a batch-1 external state broadcast over the batch, ops.py:69-75):
// a block covers 32 units x 8 batch slices; slice s walks rows s, s+8, ... and
// the broadcast state's batch sum is reduced over the 8 slices in fixed order
// (deterministic, no atomics).  Otherwise one thread per (cell, row, unit).
template <int M, bool kLoopBatch>
__global__ void __launch_bounds__(256) cell_bwd_kernel(CellArgs a) {
  pdl_prologue();
  const CellSlots S(M);
  __shared__ float red[M > 0 ? M : 1][8][32];
  __shared__ const float* sv[20];
  __shared__ float* sd[20];
  const int64_t per = kLoopBatch ? (int64_t)((a.H + 31) / 32) * 256 : (int64_t)a.batch * a.H;
  const int bpc = (int)((per + 255) / 256);
  const int j = blockIdx.x / bpc;
  if ((int)threadIdx.x < a.nslot) {
    sv[threadIdx.x] = a.val[(int64_t)threadIdx.x * a.n + j];
    sd[threadIdx.x] = a.grad[(int64_t)threadIdx.x * a.n + j];
  }
  __syncthreads();
  {
    const int64_t q = (int64_t)(blockIdx.x % bpc) * 256 + threadIdx.x;
    if (!kLoopBatch && q >= per) return;
    auto V = [&](int slot) { return sv[slot]; };
    auto D = [&](int slot) { return sd[slot]; };
    int b_lo, b_hi, b_step, u;
    if (kLoopBatch) {
      const int slice = threadIdx.x >> 5;
      u = static_cast<int>(q / 256) * 32 + (threadIdx.x & 31);
      b_lo = slice;
      b_hi = u < a.H ? a.batch : 0;
      b_step = 8;
    } else {
      b_lo = static_cast<int>(q / a.H);
      b_hi = b_lo + 1;
      b_step = 1;
      u = static_cast<int>(q - (int64_t)b_lo * a.H);
    }
    float acc_c[M > 0 ? M : 1];
#pragma unroll
    for (int k = 0; k < M; ++k) acc_c[k] = 0.f;
    for (int b = b_lo; b < b_hi; b += b_step) {
      const int64_t r = (int64_t)b * a.H + u;
      float* dG = D(0) + (int64_t)b * a.gw;
      // every load first: the slots are distinct nodes, but the compiler
      // cannot know, so a load after a store to another slot would wait for
      // the store (one L2 round trip per read-modify-write otherwise)
      const float gh = D(S.h)[r];
      const float ao = V(S.act0 + S.go())[r], ai = V(S.act0 + S.gi())[r], ag = V(S.act0 + S.gg())[r];
      const float tc = V(S.tc)[r];
      const float dc_ext = D(S.c)[r];
      const float o_tc = D(S.tc)[r], o_ao = D(S.act0 + S.go())[r], o_ai = D(S.act0 + S.gi())[r];
      const float o_ag = D(S.act0 + S.gg())[r];
      const float o_pi = D(S.pick0 + S.gi())[r], o_po = D(S.pick0 + S.go())[r], o_pg = D(S.pick0 + S.gg())[r];
      const float o_gi = dG[a.off_i + u], o_go = dG[a.off_o + u], o_gg = dG[a.off_g + u];
      const float o_p0 = M > 0 ? D(S.prod0)[r] : 0.f;
      float o_add[M > 1 ? M - 1 : 1], o_pk[M > 0 ? M : 1], o_af[M > 0 ? M : 1], o_pf[M > 0 ? M : 1];
      float o_gf[M > 0 ? M : 1], ck[M > 0 ? M : 1], af[M > 0 ? M : 1], o_ck[M > 0 ? M : 1];
#pragma unroll
      for (int k = 0; k + 1 < M; ++k) o_add[k] = D(S.add0 + k)[r];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const int64_t rc = a.cext_b1[k] ? u : r;
        o_pk[k] = D(S.prod0 + 1 + k)[r];
        ck[k] = V(1 + k)[rc];
        af[k] = V(S.act0 + S.gf(k))[r];
        o_af[k] = D(S.act0 + S.gf(k))[r];
        o_pf[k] = D(S.pick0 + S.gf(k))[r];
        o_gf[k] = dG[a.off_f[k] + u];
        o_ck[k] = (kLoopBatch && a.cext_b1[k]) ? 0.f : D(1 + k)[rc];
      }
      // h = o * tanh(c); c slot: external contributions + tanh path
      const float d_tc = gh * ao;
      const float d_o = gh * tc;
      const float dc = dc_ext + (1.f - tc * tc) * d_tc;
      // i * g
      const float d_i = dc * ag, d_g = dc * ai;
      const float dpi = ai * (1.f - ai) * d_i;
      const float dpo = ao * (1.f - ao) * d_o;
      const float dpg = (1.f - ag * ag) * d_g;
      D(S.tc)[r] = o_tc + d_tc;
      D(S.act0 + S.go())[r] = o_ao + d_o;
      D(S.c)[r] = dc;
#pragma unroll
      for (int k = 0; k + 1 < M; ++k) D(S.add0 + k)[r] = o_add[k] + dc;
      if (M > 0) D(S.prod0)[r] = o_p0 + dc;
      D(S.act0 + S.gi())[r] = o_ai + d_i;
      D(S.act0 + S.gg())[r] = o_ag + d_g;
      D(S.pick0 + S.gi())[r] = o_pi + dpi;
      D(S.pick0 + S.go())[r] = o_po + dpo;
      D(S.pick0 + S.gg())[r] = o_pg + dpg;
      dG[a.off_i + u] = o_gi + dpi;
      dG[a.off_o + u] = o_go + dpo;
      dG[a.off_g + u] = o_gg + dpg;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        D(S.prod0 + 1 + k)[r] = o_pk[k] + dc;
        const int64_t rc = a.cext_b1[k] ? u : r;
        const float d_f = dc * ck[k];
        const float d_ck = dc * af[k];
        D(S.act0 + S.gf(k))[r] = o_af[k] + d_f;
        const float dpf = af[k] * (1.f - af[k]) * d_f;
        D(S.pick0 + S.gf(k))[r] = o_pf[k] + dpf;
        dG[a.off_f[k] + u] = o_gf[k] + dpf;
        if (kLoopBatch && a.cext_b1[k]) acc_c[k] += d_ck;
        else D(1 + k)[rc] = o_ck[k] + d_ck;
      }
    }
    if (kLoopBatch) {
      const int slice = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
      for (int k = 0; k < M; ++k) red[k][slice][lane] = acc_c[k];
      __syncthreads();
      if (slice == 0 && u < a.H) {
#pragma unroll
        for (int k = 0; k < M; ++k) {
          if (!a.cext_b1[k]) continue;
          float s = 0.f;
#pragma unroll
          for (int w = 0; w < 8; ++w) s += red[k][w][lane];
          D(1 + k)[u] += s;
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- GRU parts
// (kernels.cuh GruArgs).  Arithmetic node by node as the generic kernels:
// logistic = sigmoidf_ref, scalar_mul x * c, add a + b, cmult a * b, tanhf;
// backward accumulations in the reference's reverse node order.
template <bool kB>
__global__ void __launch_bounds__(256) gru_fwd_kernel(GruArgs a) {
  pdl_prologue();
  const int64_t per = (int64_t)a.batch * a.H;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < per * a.n; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / per);
    const int64_t r = t - (int64_t)j * per;
    const int b = static_cast<int>(r / a.H), u = static_cast<int>(r - (int64_t)b * a.H);
    auto V = [&](int slot) { return const_cast<float*>(a.val[(int64_t)slot * a.n + j]); };
    const int64_t rg = (int64_t)b * a.gw;
    const int64_t rh_ = a.h_b1 ? u : r;
    if (!kB) {
      const float* zr = V(0);
      const float* ax = V(1);
      const float pz = zr[rg + a.off0 + u], pr = zr[rg + a.off1 + u], cx = ax[rg + a.off2 + u];
      const float h = V(2)[rh_];
      const float z = sigmoidf_ref(pz), rr = sigmoidf_ref(pr);
      V(3)[r] = pz;
      V(4)[r] = z;
      V(5)[r] = pr;
      V(6)[r] = rr;
      V(7)[r] = cx;
      V(8)[r] = rr * h;
    } else {
      const float ch = V(0)[rg + a.off0 + u];
      const float cx = V(1)[r], z = V(2)[r], ones = V(3)[a.ones_b1 ? u : r], h = V(4)[rh_];
      const float sv = cx + ch;
      const float cand = tanhf(sv);
      const float nz = z * -1.f;
      const float keep = ones + nz;
      const float kh = keep * h, zc = z * cand;
      V(5)[r] = ch;
      V(6)[r] = sv;
      V(7)[r] = cand;
      V(8)[r] = nz;
      V(9)[r] = keep;
      V(10)[r] = kh;
      V(11)[r] = zc;
      V(12)[r] = kh + zc;
    }
  }
}

template <bool kB>
__global__ void __launch_bounds__(256) gru_bwd_kernel(GruArgs a) {
  pdl_prologue();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)a.n * a.H;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / a.H), u = static_cast<int>(t - (int64_t)j * a.H);
    auto V = [&](int slot) { return a.val[(int64_t)slot * a.n + j]; };
    auto D = [&](int slot) { return a.grad[(int64_t)slot * a.n + j]; };
    float acc_h = 0.f, acc_ones = 0.f;
    for (int b = 0; b < a.batch; ++b) {
      const int64_t r = (int64_t)b * a.H + u, rg = (int64_t)b * a.gw;
      const int64_t rh_ = a.h_b1 ? u : r;
      if (!kB) {
        // loads first (no store-to-load waits)
        const float h = V(2)[rh_], z = V(4)[r], rr = V(6)[r];
        const float g_pz = D(3)[r], g_z = D(4)[r], g_pr = D(5)[r], g_r = D(6)[r], g_cx = D(7)[r], g_rh = D(8)[r];
        const float o_zr0 = D(0)[rg + a.off0 + u], o_zr1 = D(0)[rg + a.off1 + u], o_ax = D(1)[rg + a.off2 + u];
        const float o_h = a.h_b1 ? 0.f : D(2)[r];
        // rh = r * h
        const float gr_tot = g_r + g_rh * h;
        const float dh = g_rh * rr;
        // cx = pick(ax); r = logistic(pr); pr = pick(zr); z = logistic(pz); pz = pick(zr)
        const float gpr_tot = g_pr + rr * (1.f - rr) * gr_tot;
        const float gpz_tot = g_pz + z * (1.f - z) * g_z;
        D(6)[r] = gr_tot;
        D(5)[r] = gpr_tot;
        D(3)[r] = gpz_tot;
        D(1)[rg + a.off2 + u] = o_ax + g_cx;
        D(0)[rg + a.off1 + u] = o_zr1 + gpr_tot;
        D(0)[rg + a.off0 + u] = o_zr0 + gpz_tot;
        if (a.h_b1) acc_h += dh;
        else D(2)[r] = o_h + dh;
      } else {
        const float h = V(4)[rh_], z = V(2)[r], cand = V(7)[r], keep = V(9)[r];
        const float g_nh = D(12)[r];
        const float o_zc = D(11)[r], o_kh = D(10)[r], o_keep = D(9)[r], o_nz = D(8)[r], o_cand = D(7)[r];
        const float o_s = D(6)[r], o_ch = D(5)[r], o_z = D(2)[r], o_cx = D(1)[r];
        const float o_mh = D(0)[rg + a.off0 + u];
        const float o_ones = a.ones_b1 ? 0.f : D(3)[r];
        const float o_h = a.h_b1 ? 0.f : D(4)[r];
        // nh = kh + zc
        const float g_zc = o_zc + g_nh, g_kh = o_kh + g_nh;
        // zc = z * cand
        float gz = o_z + g_zc * cand;
        const float g_cand = o_cand + g_zc * z;
        // kh = keep * h
        const float g_keep = o_keep + g_kh * h;
        const float dh = g_kh * keep;
        // keep = ones + nz
        const float dones = g_keep;
        const float g_nz = o_nz + g_keep;
        // nz = z * -1
        gz = gz + -1.f * g_nz;
        // cand = tanh(s); s = cx + ch; ch = pick(mh)
        const float g_s = o_s + (1.f - cand * cand) * g_cand;
        const float g_ch = o_ch + g_s;
        D(11)[r] = g_zc;
        D(10)[r] = g_kh;
        D(9)[r] = g_keep;
        D(8)[r] = g_nz;
        D(7)[r] = g_cand;
        D(6)[r] = g_s;
        D(5)[r] = g_ch;
        D(2)[r] = gz;
        D(1)[r] = o_cx + g_s;
        D(0)[rg + a.off0 + u] = o_mh + g_ch;
        if (a.ones_b1) acc_ones += dones;
        else D(3)[r] = o_ones + dones;
        if (a.h_b1) acc_h += dh;
        else D(4)[r] = o_h + dh;
      }
    }
    if (a.h_b1) D(kB ? 4 : 2)[u] += acc_h;
    if (kB && a.ones_b1) D(3)[u] += acc_ones;
  }
}

// ------------------------------------------------------------------ structural

__global__ void pick_fwd_kernel(PickArgs a) {
  pdl_prologue();
  const int64_t per = (int64_t)a.batch * a.width;
  const int64_t total = per * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / per);
    const int64_t r = t - (int64_t)j * per;
    const int64_t b = r / a.width, e = r - b * a.width;
    a.out[j][r] = a.in[j][b * a.in_elem + a.lo + e];
  }
}

__global__ void pick_bwd_kernel(PickArgs a) {
  pdl_prologue();
  const int64_t per = (int64_t)a.batch * a.width;
  const int64_t total = per * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / per);
    const int64_t r = t - (int64_t)j * per;
    const int64_t b = r / a.width, e = r - b * a.width;
    a.gin[j][b * a.in_elem + a.lo + e] += a.gout[j][r];
  }
}

__device__ __forceinline__ int find_part(const int* offs, int parts, int col) {
  int k = 0;
  while (k + 1 < parts && col >= offs[k + 1]) ++k;
  return k;
}

__global__ void concat_fwd_kernel(ConcatArgs a) {
  pdl_prologue();
  const int64_t per = (int64_t)a.batch * a.total;
  const int64_t all = per * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < all; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / per);
    const int64_t r = t - (int64_t)j * per;
    const int b = static_cast<int>(r / a.total), col = static_cast<int>(r - (int64_t)b * a.total);
    const int k = find_part(a.offs, a.parts, col);
    const int w = a.offs[k + 1] - a.offs[k];
    a.out[j][r] = a.in[(int64_t)k * a.n + j][(int64_t)b * w + (col - a.offs[k])];
  }
}

__global__ void concat_bwd_kernel(ConcatArgs a) {
  pdl_prologue();
  const int64_t per = (int64_t)a.batch * a.total;
  const int64_t all = per * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < all; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / per);
    const int64_t r = t - (int64_t)j * per;
    const int b = static_cast<int>(r / a.total), col = static_cast<int>(r - (int64_t)b * a.total);
    const int k = find_part(a.offs, a.parts, col);
    const int w = a.offs[k + 1] - a.offs[k];
    a.gin[(int64_t)k * a.n + j][(int64_t)b * w + (col - a.offs[k])] += a.gout[j][r];
  }
}

__global__ void sum_batches_fwd_kernel(SumBatchesArgs a) {
  pdl_prologue();
  const int64_t total = (int64_t)a.elem * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / a.elem);
    const int e = static_cast<int>(t - (int64_t)j * a.elem);
    // 16 loads in flight, added in batch order
    const float* src = a.in[j] + e;
    float s = 0.f;
    int b = 0;
    for (; b + 16 <= a.batch; b += 16) {
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = src[(int64_t)(b + q) * a.elem];
#pragma unroll
      for (int q = 0; q < 16; ++q) s += v[q];
    }
    for (; b < a.batch; ++b) s += src[(int64_t)b * a.elem];
    a.out[j][e] = s;
  }
}

__global__ void sum_batches_bwd_kernel(SumBatchesArgs a) {
  pdl_prologue();
  const int64_t per = (int64_t)a.batch * a.elem;
  const int64_t total = per * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(t / per);
    const int64_t r = t - (int64_t)j * per;
    a.gin[j][r] += a.gout[j][r % a.elem];
  }
}

// ------------------------------------------------------------------ row-wise
// One warp per row for narrow rows, one 256-thread block per row otherwise.

template <bool kBlock>
__device__ __forceinline__ float row_reduce_max(float v, float* sh) {
  v = warp_max(v);
  if (!kBlock) return v;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : -INFINITY;
  if (w == 0) {
    r = warp_max(r);
    if (lane == 0) sh[0] = r;
  }
  __syncthreads();
  return sh[0];
}

template <bool kBlock>
__device__ __forceinline__ float row_reduce_sum(float v, float* sh) {
  v = warp_sum(v);
  if (!kBlock) return v;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.f;
  if (w == 0) {
    r = warp_sum(r);
    if (lane == 0) sh[0] = r;
  }
  __syncthreads();
  return sh[0];
}

// op: 0 softmax fwd, 1 softmax bwd, 2 pnls fwd, 3 pnls bwd
template <int kOp, bool kBlock>
__global__ void row_kernel(RowArgs a) {
  pdl_prologue();
  __shared__ float sh[32];
  const int row = kBlock ? blockIdx.x : (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (row >= a.rows) return;
  const int stride = kBlock ? blockDim.x : 32;
  const int tid = kBlock ? threadIdx.x : (threadIdx.x & 31);
  const int j = row / a.batch, b = row - j * a.batch;
  const int64_t off = (int64_t)b * a.width;
  if (kOp == 1) {  // softmax backward: gin += y * (g - <g, y>)   (ops.py:240-247)
    const float* y = a.oval[j] + off;
    const float* g = a.gout[j] + off;
    float d = 0.f;
    for (int c = tid; c < a.width; c += stride) d += g[c] * y[c];
    d = row_reduce_sum<kBlock>(d, sh);
    float* gi = a.gin[j] + off;
    for (int c = tid; c < a.width; c += stride) gi[c] += y[c] * (g[c] - d);
    return;
  }
  const float* x = a.in[j] + off;
  float m = -INFINITY;
  for (int c = tid; c < a.width; c += stride) m = fmaxf(m, x[c]);
  m = row_reduce_max<kBlock>(m, sh);
  float s = 0.f;
  for (int c = tid; c < a.width; c += stride) s += expf(x[c] - m);
  s = row_reduce_sum<kBlock>(s, sh);
  if (kOp == 0) {  // softmax forward (ops.py:231-237)
    float* o = a.out[j] + off;
    for (int c = tid; c < a.width; c += stride) o[c] = expf(x[c] - m) / s;
  } else if (kOp == 2) {  // pnls forward: max + log sum exp(x - max) - x[label] (ops.py:470-473)
    if (tid == 0) a.out[j][b] = m + logf(s) - x[a.labels[row]];
  } else {  // pnls backward: gin += g * (softmax - onehot) (ops.py:476-479, 503-508)
    const float g = a.gout[j][b];
    const int lab = a.labels[row];
    float* gi = a.gin[j] + off;
    for (int c = tid; c < a.width; c += stride) {
      float p = expf(x[c] - m) / s;
      if (c == lab) p -= 1.f;
      gi[c] = (a.overwrite ? 0.f : gi[c]) + g * p;
    }
  }
}

// Wide rows (softmax / pnls over a vocabulary): one 256-thread block per row
// with the row held in registers (kV float4 per thread), so x is read from
// memory once: max, sum of exp and the output pass all run from registers.
// Rows that are not 16 B aligned take the strided path above.
template <int kOp, int kV>
__global__ void __launch_bounds__(256) row_reg_kernel(RowArgs a) {
  pdl_prologue();
  __shared__ float sh[32];
  const int row = blockIdx.x;
  const int j = row / a.batch, b = row - j * a.batch;
  const int64_t off = (int64_t)b * a.width;
  const float* x = a.in[j] + off;
  float* gi = kOp == 3 ? a.gin[j] + off : nullptr;
  float* o = kOp == 0 ? a.out[j] + off : nullptr;
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(gi) |
                         reinterpret_cast<uintptr_t>(o)) & 15) == 0;
  if (!aligned) {  // block-uniform
    const int tid = threadIdx.x;
    float m = -INFINITY;
    for (int c = tid; c < a.width; c += 256) m = fmaxf(m, x[c]);
    m = row_reduce_max<true>(m, sh);
    float s = 0.f;
    for (int c = tid; c < a.width; c += 256) s += expf(x[c] - m);
    s = row_reduce_sum<true>(s, sh);
    if (kOp == 0) {
      for (int c = tid; c < a.width; c += 256) o[c] = expf(x[c] - m) / s;
    } else if (kOp == 2) {
      if (tid == 0) a.out[j][b] = m + logf(s) - x[a.labels[row]];
    } else {
      const float g = a.gout[j][b];
      const int lab = a.labels[row];
      for (int c = tid; c < a.width; c += 256) {
        float p = expf(x[c] - m) / s;
        if (c == lab) p -= 1.f;
        gi[c] = (a.overwrite ? 0.f : gi[c]) + g * p;
      }
    }
    return;
  }
  const int n4 = a.width >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4 v[kV];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int q = threadIdx.x + 256 * i;
    v[i] = q < n4 ? x4[q] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    m = fmaxf(m, fmaxf(fmaxf(v[i].x, v[i].y), fmaxf(v[i].z, v[i].w)));
  }
  m = row_reduce_max<true>(m, sh);
  // exp(x - m) once: kept in the row registers for the output pass
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kV; ++i)
    if (threadIdx.x + 256 * i < n4) {
      v[i] = make_float4(expf(v[i].x - m), expf(v[i].y - m), expf(v[i].z - m), expf(v[i].w - m));
      s += v[i].x + v[i].y + v[i].z + v[i].w;
    }
  s = row_reduce_sum<true>(s, sh);
  if (kOp == 2) {
    if (threadIdx.x == 0) a.out[j][b] = m + logf(s) - x[a.labels[row]];
    return;
  }
  const float inv_s = 1.f / s;
  const float g = kOp == 3 ? a.gout[j][b] : 1.f;
  const int lab = kOp == 3 ? a.labels[row] : -1;
  float4* d4 = reinterpret_cast<float4*>(kOp == 3 ? gi : o);
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    const int q = threadIdx.x + 256 * i;
    if (q >= n4) continue;
    float4 p = make_float4(v[i].x * inv_s, v[i].y * inv_s, v[i].z * inv_s, v[i].w * inv_s);
    if (kOp == 3) {
      if ((lab >> 2) == q) {
        const int e = lab & 3;
        if (e == 0) p.x -= 1.f;
        else if (e == 1) p.y -= 1.f;
        else if (e == 2) p.z -= 1.f;
        else p.w -= 1.f;
      }
      float4 d = a.overwrite ? make_float4(0.f, 0.f, 0.f, 0.f) : d4[q];
      d.x += g * p.x;
      d.y += g * p.y;
      d.z += g * p.z;
      d.w += g * p.w;
      d4[q] = d;
    } else {
      d4[q] = p;
    }
  }
}

// ------------------------------------------------------ two-level softmax term
// (kernels.cuh Pnls2Args): the row_kernel arithmetic (max, sum of expf(x - m),
// m + logf(s) - x[label]) for both rows of a unit, one block per unit.
__device__ __forceinline__ void row_stats(const float* x, int w, float* sh, float& m, float& s) {
  float mm = -INFINITY;
  for (int c = threadIdx.x; c < w; c += blockDim.x) mm = fmaxf(mm, x[c]);
  m = row_reduce_max<true>(mm, sh);
  float ss = 0.f;
  for (int c = threadIdx.x; c < w; c += blockDim.x) ss += expf(x[c] - m);
  s = row_reduce_sum<true>(ss, sh);
}

__global__ void __launch_bounds__(256) pnls2_fwd_kernel(Pnls2Args a) {
  pdl_prologue();
  __shared__ float sh[32];
  const int j = blockIdx.x;
  float loss[2];
  for (int k = 0; k < 2; ++k) {
    const float* x = a.val[(int64_t)k * a.n + j];
    float m, s;
    row_stats(x, a.width[2 * j + k], sh, m, s);
    loss[k] = m + logf(s) - x[a.label[2 * j + k]];
  }
  if (threadIdx.x == 0) {
    const_cast<float*>(a.val[(int64_t)2 * a.n + j])[0] = loss[0];
    const_cast<float*>(a.val[(int64_t)3 * a.n + j])[0] = loss[1];
    const_cast<float*>(a.val[(int64_t)4 * a.n + j])[0] = loss[0] + loss[1];
  }
}

__global__ void __launch_bounds__(256) pnls2_bwd_kernel(Pnls2Args a) {
  pdl_prologue();
  __shared__ float sh[32];
  const int j = blockIdx.x;
  const float gs = a.grad[(int64_t)4 * a.n + j][0];
  for (int k = 0; k < 2; ++k) {
    // the pnls node's gradient: its own slot (other consumers) + the add's
    float* gp = a.grad[(int64_t)(2 + k) * a.n + j];
    const float g = gp[0] + gs;
    const float* x = a.val[(int64_t)k * a.n + j];
    float* gx = a.grad[(int64_t)k * a.n + j];
    const int w = a.width[2 * j + k], lab = a.label[2 * j + k];
    float m, s;
    row_stats(x, w, sh, m, s);
    for (int c = threadIdx.x; c < w; c += blockDim.x) {
      float p = expf(x[c] - m) / s;
      if (c == lab) p -= 1.f;
      gx[c] += g * p;
    }
    __syncthreads();  // every thread read gp[0] before it is overwritten
    if (threadIdx.x == 0) gp[0] = g;
  }
}

template <int kOp>
int launch_rows(const RowArgs& a, cudaStream_t s) {
  if (a.rows <= 0) return 0;
  if (a.width > 512 && (a.width & 3) == 0 && a.width <= 256 * 4 * 16 && kOp != 1) {
    const int need = (a.width / 4 + 255) / 256;
    if (need <= 4) launch_k(row_reg_kernel<kOp, 4>, a.rows, 256, 0, s, a);
    else if (need <= 8) launch_k(row_reg_kernel<kOp, 8>, a.rows, 256, 0, s, a);
    else if (need <= 12) launch_k(row_reg_kernel<kOp, 12>, a.rows, 256, 0, s, a);
    else launch_k(row_reg_kernel<kOp, 16>, a.rows, 256, 0, s, a);
  } else if (a.width > 512) {
    launch_k(row_kernel<kOp, true>, a.rows, 256, 0, s, a);
  } else {
    const int rows_per_block = 8;
    launch_k(row_kernel<kOp, false>, (a.rows + rows_per_block - 1) / rows_per_block, 32 * rows_per_block, 0, s, a);
  }
  return 1;
}

// ------------------------------------------------------------- lookup tables

__global__ void gather_rows_kernel(const float* __restrict__ table, int dim, const int64_t* __restrict__ ids,
                                   float* const* out_rows, int rows) {
  pdl_prologue();
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= rows) return;
  const int lane = threadIdx.x & 31;
  const float* src = table + ids[w] * (int64_t)dim;
  float* dst = out_rows[w];
  const bool vec = ((dim & 3) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  if (vec) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int c = lane; c < (dim >> 2); c += 32) d4[c] = __ldg(s4 + c);
  } else {
    for (int c = lane; c < dim; c += 32) dst[c] = src[c];
  }
}

// Sorted segmented scatter of lookup-row gradients (graph.py:57-63
// `np.add.at`), deterministic and atomic-free in its arithmetic: one warp per
// work item; a segment of <= kScatterChunk rows is one item that writes its
// row directly; a longer segment (the EOS padding id collects one row per
// padded position) is split into chunks whose partial sums go to scratch, and
// the warp that finishes a segment's last chunk (arrival counter) adds the
// partials in chunk order.  Rows are summed in segment order inside a chunk,
// 8 row loads in flight per lane.
template <bool kSet>
__global__ void __launch_bounds__(256) scatter_rows_kernel(float* __restrict__ table_grad, int dim,
                                                           const int64_t* __restrict__ ids,
                                                           const ScatterItem* __restrict__ items, int n_items,
                                                           const float* const* __restrict__ src_rows,
                                                           float* __restrict__ partials, int* __restrict__ counters,
                                                           float scale) {
  pdl_prologue();
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (w >= n_items) return;
  const int lane = threadIdx.x & 31;
  const ScatterItem it = items[w];
  float* dst = table_grad + ids[it.u] * (int64_t)dim;
  const bool chunked = it.nchunks > 0;
  float* part = chunked ? partials + (int64_t)(it.pbase + it.chunk) * dim : nullptr;
  // the item's <= kScatterChunk row pointers in one round of independent
  // loads, then every row's data in flight at once (two memory round trips
  // per item); alignment decided from the loaded pointers
  const int nk = it.k1 - it.k0;
  const float* rp[kScatterChunk];
  bool vec = (dim & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
#pragma unroll
  for (int r = 0; r < kScatterChunk; ++r) {
    rp[r] = r < nk ? src_rows[it.k0 + r] : nullptr;
    if (r < nk) vec = vec && (reinterpret_cast<uintptr_t>(rp[r]) & 15) == 0;
  }
  auto finish = [&](int c, float s) {
    if (chunked) {
      part[c] = s;
    } else if (kSet) {
      dst[c] = s / scale;
    } else {
      dst[c] += scale * s;
    }
  };
  if (vec) {
    for (int c4 = lane; c4 < (dim >> 2); c4 += 32) {
      float4 v[kScatterChunk];
#pragma unroll
      for (int r = 0; r < kScatterChunk; ++r)
        v[r] = r < nk ? __ldg(reinterpret_cast<const float4*>(rp[r]) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < kScatterChunk; ++r)
        if (r < nk) {
          acc.x += v[r].x;
          acc.y += v[r].y;
          acc.z += v[r].z;
          acc.w += v[r].w;
        }
      finish(4 * c4 + 0, acc.x);
      finish(4 * c4 + 1, acc.y);
      finish(4 * c4 + 2, acc.z);
      finish(4 * c4 + 3, acc.w);
    }
  } else {
    for (int c = lane; c < dim; c += 32) {
      float acc = 0.f;
      for (int r = 0; r < nk; ++r) acc += rp[r][c];
      finish(c, acc);
    }
  }
  if (!chunked) return;
  // last chunk of the segment to arrive combines the partials in chunk order
  __threadfence();
  int last = 0;
  if (lane == 0) last = atomicAdd(counters + it.seg_slot, 1) == it.nchunks - 1;
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  const float* pb = partials + (int64_t)it.pbase * dim;
  if ((dim & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (reinterpret_cast<uintptr_t>(pb) & 15) == 0) {
    // one float4 column group per lane, 16 partial loads in flight (the EOS
    // segment of a padded minibatch has ~60 chunks); same chunk-order sums
    for (int c4 = lane; c4 < (dim >> 2); c4 += 32) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q0 = 0; q0 < it.nchunks; q0 += 16) {
        float4 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (q0 + i < it.nchunks) v[i] = __ldcg(reinterpret_cast<const float4*>(pb + (int64_t)(q0 + i) * dim) + c4);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (q0 + i < it.nchunks) {
            s.x += v[i].x;
            s.y += v[i].y;
            s.z += v[i].z;
            s.w += v[i].w;
          }
      }
      float* d = dst + 4 * c4;
      if (kSet) {
        d[0] = s.x / scale, d[1] = s.y / scale, d[2] = s.z / scale, d[3] = s.w / scale;
      } else {
        d[0] += scale * s.x, d[1] += scale * s.y, d[2] += scale * s.z, d[3] += scale * s.w;
      }
    }
    if (lane == 0) counters[it.seg_slot] = 0;
    return;
  }
  for (int c = lane; c < dim; c += 32) {
    float s = 0.f;
    int q = 0;
    for (; q + 8 <= it.nchunks; q += 8) {  // 8 partial loads in flight, summed in chunk order
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldcg(pb + (int64_t)(q + i) * dim + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) s += v[i];
    }
    for (; q < it.nchunks; ++q) s += __ldcg(pb + (int64_t)q * dim + c);
    if (kSet) {
      dst[c] = s / scale;
    } else {
      dst[c] += scale * s;
    }
  }
  if (lane == 0) counters[it.seg_slot] = 0;  // left at zero for the next launch
}

__global__ void pack_rows_kernel(const float* __restrict__ table, int dim, const int64_t* __restrict__ ids,
                                 float* __restrict__ out, int n) {
  pdl_prologue();
  const int64_t total = (int64_t)n * dim;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = t / dim, c = t - u * dim;
    out[t] = table[ids[u] * dim + c];
  }
}

// ------------------------------------------------------------------ generic

// matmul per batch element, column-major: out(i,c) = sum_t A(i,t) X(t,c)
__global__ void matmul_fwd_kernel(MatmulArgs a) {
  pdl_prologue();
  const int64_t osz = (int64_t)a.m * a.p;
  const int64_t total = osz * a.batch * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jb = t / osz;
    const int64_t o = t - jb * osz;
    const int j = static_cast<int>(jb / a.batch), b = static_cast<int>(jb - (int64_t)j * a.batch);
    const int i = static_cast<int>(o % a.m), c = static_cast<int>(o / a.m);
    const float* A = a.a[j] + (a.a_b1 ? 0 : (int64_t)b * a.m * a.k);
    const float* X = a.x[j] + (a.x_b1 ? 0 : (int64_t)b * a.k * a.p);
    float s = 0.f;
    for (int q = 0; q < a.k; ++q) s += A[i + (int64_t)q * a.m] * X[q + (int64_t)c * a.k];
    a.out[j][(int64_t)b * osz + o] = s;
  }
}

// gA(i,q) += sum_b sum_c g(i,c) X(q,c);  one thread per (node, A-batch, element)
__global__ void matmul_bwd_a_kernel(MatmulArgs a) {
  pdl_prologue();
  const int ab = a.a_b1 ? 1 : a.batch;
  const int64_t asz = (int64_t)a.m * a.k;
  const int64_t total = asz * ab * a.n;
  const int64_t osz = (int64_t)a.m * a.p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jb = t / asz;
    const int64_t o = t - jb * asz;
    const int j = static_cast<int>(jb / ab), bb = static_cast<int>(jb - (int64_t)j * ab);
    const int i = static_cast<int>(o % a.m), q = static_cast<int>(o / a.m);
    float s = 0.f;
    const int b0 = a.a_b1 ? 0 : bb, b1 = a.a_b1 ? a.batch : bb + 1;
    for (int b = b0; b < b1; ++b) {
      const float* X = a.x[j] + (a.x_b1 ? 0 : (int64_t)b * a.k * a.p);
      const float* G = a.gout[j] + (int64_t)b * osz;
      for (int c = 0; c < a.p; ++c) s += G[i + (int64_t)c * a.m] * X[q + (int64_t)c * a.k];
    }
    a.ga[j][(int64_t)bb * asz + o] += s;
  }
}

// gX(q,c) += sum_b sum_i A(i,q) g(i,c)
__global__ void matmul_bwd_x_kernel(MatmulArgs a) {
  pdl_prologue();
  const int xb = a.x_b1 ? 1 : a.batch;
  const int64_t xsz = (int64_t)a.k * a.p;
  const int64_t total = xsz * xb * a.n;
  const int64_t osz = (int64_t)a.m * a.p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jb = t / xsz;
    const int64_t o = t - jb * xsz;
    const int j = static_cast<int>(jb / xb), bb = static_cast<int>(jb - (int64_t)j * xb);
    const int q = static_cast<int>(o % a.k), c = static_cast<int>(o / a.k);
    float s = 0.f;
    const int b0 = a.x_b1 ? 0 : bb, b1 = a.x_b1 ? a.batch : bb + 1;
    for (int b = b0; b < b1; ++b) {
      const float* A = a.a[j] + (a.a_b1 ? 0 : (int64_t)b * a.m * a.k);
      const float* G = a.gout[j] + (int64_t)b * osz;
      for (int i = 0; i < a.m; ++i) s += A[i + (int64_t)q * a.m] * G[i + (int64_t)c * a.m];
    }
    a.gx[j][(int64_t)bb * xsz + o] += s;
  }
}

__global__ void affine_generic_fwd_kernel(AffineGenericArgs a) {
  pdl_prologue();
  const int64_t total = (int64_t)a.m * a.batch * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jb = t / a.m;
    const int i = static_cast<int>(t - jb * a.m);
    const int j = static_cast<int>(jb / a.batch), b = static_cast<int>(jb - (int64_t)j * a.batch);
    float s = a.bias[j][(a.b_b1 ? 0 : (int64_t)b * a.m) + i];
    for (int k = 0; k < a.terms; ++k) {
      const int K = a.kdim[k];
      const float* W = a.w[(int64_t)k * a.n + j] + (a.w_b1[k] ? 0 : (int64_t)b * a.m * K);
      const float* X = a.x[(int64_t)k * a.n + j] + (a.x_b1[k] ? 0 : (int64_t)b * K);
      float acc = 0.f;
      for (int q = 0; q < K; ++q) acc += W[i + (int64_t)q * a.m] * X[q];
      s += acc;
    }
    a.out[j][(int64_t)b * a.m + i] = s;
  }
}

// which: 0 bias, 1 W of term k, 2 x of term k
__global__ void affine_generic_bwd_kernel(AffineGenericArgs a, int which, int k) {
  pdl_prologue();
  const int K = which == 0 ? 1 : a.kdim[k];
  int ob;  // operand batch
  int64_t osz;
  if (which == 0) { ob = a.b_b1 ? 1 : a.batch; osz = a.m; }
  else if (which == 1) { ob = a.w_b1[k] ? 1 : a.batch; osz = (int64_t)a.m * K; }
  else { ob = a.x_b1[k] ? 1 : a.batch; osz = K; }
  const bool b1 = ob == 1 && a.batch > 1;
  const int64_t total = osz * ob * a.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jb = t / osz;
    const int64_t o = t - jb * osz;
    const int j = static_cast<int>(jb / ob), bb = static_cast<int>(jb - (int64_t)j * ob);
    const int b0 = b1 ? 0 : bb, b1e = b1 ? a.batch : bb + 1;
    float s = 0.f;
    for (int b = b0; b < b1e; ++b) {
      const float* G = a.gout[j] + (int64_t)b * a.m;
      if (which == 0) {
        s += G[o];
      } else if (which == 1) {
        const int i = static_cast<int>(o % a.m), q = static_cast<int>(o / a.m);
        const float* X = a.x[(int64_t)k * a.n + j] + (a.x_b1[k] ? 0 : (int64_t)b * K);
        s += G[i] * X[q];
      } else {
        const float* W = a.w[(int64_t)k * a.n + j] + (a.w_b1[k] ? 0 : (int64_t)b * a.m * K);
        const int q = static_cast<int>(o);
        for (int i = 0; i < a.m; ++i) s += W[i + (int64_t)q * a.m] * G[i];
      }
    }
    float* dst = which == 0 ? a.gbias[j] : (which == 1 ? a.gw[(int64_t)k * a.n + j] : a.gx[(int64_t)k * a.n + j]);
    dst[(int64_t)bb * osz + o] += s;
  }
}

// column sums over gathered rows, two deterministic passes
__global__ void colsum_partial_kernel(const float* const* rows, int n_rows, int width, int chunks, float* work) {
  pdl_prologue();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int ch = blockIdx.y;
  if (c >= width) return;
  const int r0 = (int)((int64_t)n_rows * ch / chunks), r1 = (int)((int64_t)n_rows * (ch + 1) / chunks);
  // 8 rows in flight (pointers, then values), summed in row order
  float s = 0.f;
  int r = r0;
  for (; r + 8 <= r1; r += 8) {
    const float* p[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = rows[r + k];
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = p[k][c];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; r < r1; ++r) s += rows[r][c];
  work[(int64_t)ch * width + c] = s;
}

__global__ void colsum_final_kernel(float* dst, const float* work, int width, int chunks) {
  pdl_prologue();
  // block = 32 columns x 8 chunk groups; group y sums chunks y, y+8, ...
  // (4 in flight), then the 8 group sums are added in fixed order
  __shared__ float part[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31), y = threadIdx.x >> 5;
  float s = 0.f;
  if (c < width) {
    int ch = y;
    for (; ch + 24 < chunks; ch += 32) {
      const float a0 = work[(int64_t)ch * width + c], a1 = work[(int64_t)(ch + 8) * width + c];
      const float a2 = work[(int64_t)(ch + 16) * width + c], a3 = work[(int64_t)(ch + 24) * width + c];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; ch < chunks; ch += 8) s += work[(int64_t)ch * width + c];
  }
  part[y][threadIdx.x & 31] = s;
  __syncthreads();
  if (y == 0 && c < width) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += part[k][threadIdx.x];
    dst[c] += t;
  }
}

// the bias gradients of one backward (several widths / row sets) in one pair
// of launches: job q owns partial blocks [pb0, pb0 + xb*chunks) and final
// blocks [fb0, fb0 + ceil(width/32)); same arithmetic as the kernels above
__global__ void colsum_partial_group_kernel(const __grid_constant__ ColsumGroup G) {
  pdl_prologue();
  int q = 0;
  while (q + 1 < G.n && (int)blockIdx.x >= G.j[q + 1].pb0) ++q;
  const ColsumJob& J = G.j[q];
  const int lb = (int)blockIdx.x - J.pb0;
  const int xb = (J.width + 255) / 256;
  const int ch = lb / xb, c = (lb - ch * xb) * 256 + threadIdx.x;
  const int r0 = (int)((int64_t)J.n_rows * ch / J.chunks), r1 = (int)((int64_t)J.n_rows * (ch + 1) / J.chunks);
  // the chunk's row pointers staged in shared memory 64 at a time, then 16
  // rows in flight per thread: one memory round trip per 16 rows instead of
  // a pointer load followed by a dependent value load per 8 (summed in row
  // order, as before)
  __shared__ const float* rp[64];
  float s = 0.f;
  for (int base = r0; base < r1; base += 64) {
    const int cnt = min(64, r1 - base);
    __syncthreads();
    if ((int)threadIdx.x < cnt) rp[threadIdx.x] = J.rows[base + threadIdx.x];
    __syncthreads();
    if (c < J.width) {
      int k = 0;
      for (; k + 16 <= cnt; k += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = rp[k + i][c];
#pragma unroll
        for (int i = 0; i < 16; ++i) s += v[i];
      }
      for (; k < cnt; ++k) s += rp[k][c];
    }
  }
  if (c < J.width) J.work[(int64_t)ch * J.width + c] = s;
}

// Column sums over 16 B aligned rows (the logits bias: 10^4 columns over T*B
// rows; the gate biases): a block reads kColsumWideRows whole row segments of
// up to 2048 columns (contiguous 8 KiB, float4 per thread, 16 rows in flight)
// instead of many rows x 1 KiB fragments -- DRAM pages stay open.  Grouped:
// block -> (job, column slab, row chunk) through the jobs' pb0 offsets.
// work[chunk][c], rows summed in order.
constexpr int kColsumWideRows = 32;
__global__ void __launch_bounds__(256) colsum_wide_partial_kernel(const __grid_constant__ ColsumGroup G) {
  if (G.nowait) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  else pdl_prologue();
  int q = 0;
  while (q + 1 < G.n && (int)blockIdx.x >= G.j[q + 1].pb0) ++q;
  const ColsumJob& J = G.j[q];
  const int w4 = J.width >> 2;
  const int slabs = (w4 + 511) / 512;
  const int lb = (int)blockIdx.x - J.pb0;
  const int ch = lb / slabs, slab = lb - ch * slabs;
  __shared__ const float* rp[kColsumWideRows];
  const int r0 = ch * kColsumWideRows, nr = min(kColsumWideRows, J.n_rows - r0);
  if ((int)threadIdx.x < nr) rp[threadIdx.x] = J.rows[r0 + threadIdx.x];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int c4 = slab * 512 + i * 256 + threadIdx.x;
    if (c4 >= w4) continue;
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int rb = 0; rb < nr; rb += 16) {
      float4 v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r)
        v[r] = rb + r < nr ? __ldg(reinterpret_cast<const float4*>(rp[rb + r]) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (rb + r < nr) {
          sum.x += v[r].x;
          sum.y += v[r].y;
          sum.z += v[r].z;
          sum.w += v[r].w;
        }
    }
    reinterpret_cast<float4*>(J.work + (int64_t)ch * J.width)[c4] = sum;
  }
}

__global__ void colsum_final_group_kernel(const __grid_constant__ ColsumGroup G) {
  pdl_prologue();
  int q = 0;
  while (q + 1 < G.n && (int)blockIdx.x >= G.j[q + 1].fb0) ++q;
  const ColsumJob& J = G.j[q];
  __shared__ float part[8][33];
  const int c = ((int)blockIdx.x - J.fb0) * 32 + (threadIdx.x & 31), y = threadIdx.x >> 5;
  float s = 0.f;
  if (c < J.width) {
    int ch = y;
    for (; ch + 24 < J.chunks; ch += 32) {
      const float a0 = J.work[(int64_t)ch * J.width + c], a1 = J.work[(int64_t)(ch + 8) * J.width + c];
      const float a2 = J.work[(int64_t)(ch + 16) * J.width + c], a3 = J.work[(int64_t)(ch + 24) * J.width + c];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; ch < J.chunks; ch += 8) s += J.work[(int64_t)ch * J.width + c];
  }
  part[y][threadIdx.x & 31] = s;
  __syncthreads();
  if (y == 0 && c < J.width) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += part[k][threadIdx.x];
    J.dst[c] += t;
  }
}

__global__ void row_reduce_scatter_kernel(float* const* dst_rows, const int* seg, const float* src, int n_targets,
                                          int width) {
  pdl_prologue();
  // one block per target row; 8 warps split the segment, fixed-order reduce
  __shared__ float part[8][128];
  const int u = blockIdx.x;
  if (u >= n_targets) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* dst = dst_rows[u];
  for (int c0 = 0; c0 < width; c0 += 128) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = seg[u] + w; k < seg[u + 1]; k += 8) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + lane + 32 * q;
        if (c < width) acc[q] += src[(int64_t)k * width + c];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) part[w][lane + 32 * q] = acc[q];
    __syncthreads();
    if (threadIdx.x < 128 && c0 + threadIdx.x < width) {
      float s = 0.f;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s += part[ww][threadIdx.x];
      dst[c0 + threadIdx.x] += s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ trainers
// trainers.py:63-83 elementwise rules; the gradient is zeroed in the same pass
// (Model.zero_gradients, params.py:114-119).

__device__ __forceinline__ void apply_rule(const RuleArgs& r, float& w, float& g, float* s0, float* s1) {
  switch (r.rule) {
    case 0:
      w = w - r.lr * g;
      break;
    case 1: {
      const float v = r.momentum * (*s0) - r.lr * g;
      *s0 = v;
      w = w + v;
      break;
    }
    case 2: {
      const float sq = (*s0) + g * g;
      *s0 = sq;
      w = w - r.lr * g / (sqrtf(sq) + r.adagrad_eps);
      break;
    }
    default: {
      const float m1 = r.beta1 * (*s0) + (1.f - r.beta1) * g;
      const float m2 = r.beta2 * (*s1) + (1.f - r.beta2) * (g * g);
      *s0 = m1;
      *s1 = m2;
      const float mhat = m1 / r.bc1;
      const float vhat = m2 / r.bc2;
      w = w - r.lr * mhat / (sqrtf(vhat) + r.adam_eps);
      break;
    }
  }
  g = 0.f;
}

constexpr int kUpdChunk = 2048;

__global__ void update_dense_kernel(RuleArgs r, const TensorSeg* __restrict__ segs, int nseg) {
  pdl_prologue();
  // locate this block's segment: segments are laid out in order, each taking
  // ceil(n / kUpdChunk) blocks
  int blk = blockIdx.x, s = 0;
  for (; s < nseg; ++s) {
    const int nb = static_cast<int>((segs[s].n + kUpdChunk - 1) / kUpdChunk);
    if (blk < nb) break;
    blk -= nb;
  }
  if (s >= nseg) return;
  const TensorSeg sg = segs[s];
  const int64_t e0 = (int64_t)blk * kUpdChunk;
  const int64_t e1 = min(e0 + kUpdChunk, sg.n);
  float dummy0 = 0.f, dummy1 = 0.f;
  int64_t e_tail = e0;
  const uintptr_t al = reinterpret_cast<uintptr_t>(sg.w) | reinterpret_cast<uintptr_t>(sg.g) |
                       reinterpret_cast<uintptr_t>(sg.s0) | reinterpret_cast<uintptr_t>(sg.s1);
  if ((al & 15) == 0 && (e0 & 3) == 0) {
    // 16 B accesses: 4 parameters (w, g and the rule's state) per thread
    const int64_t n4 = (e1 - e0) >> 2;
    for (int64_t q = threadIdx.x; q < n4; q += blockDim.x) {
      const int64_t e = e0 + 4 * q;
      float4 w4 = *reinterpret_cast<const float4*>(sg.w + e), g4 = *reinterpret_cast<const float4*>(sg.g + e);
      float4 a4 = sg.s0 ? *reinterpret_cast<const float4*>(sg.s0 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 b4 = sg.s1 ? *reinterpret_cast<const float4*>(sg.s1 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      apply_rule(r, w4.x, g4.x, &a4.x, &b4.x);
      apply_rule(r, w4.y, g4.y, &a4.y, &b4.y);
      apply_rule(r, w4.z, g4.z, &a4.z, &b4.z);
      apply_rule(r, w4.w, g4.w, &a4.w, &b4.w);
      *reinterpret_cast<float4*>(sg.w + e) = w4;
      *reinterpret_cast<float4*>(sg.g + e) = g4;
      if (sg.s0) *reinterpret_cast<float4*>(sg.s0 + e) = a4;
      if (sg.s1) *reinterpret_cast<float4*>(sg.s1 + e) = b4;
    }
    e_tail = e0 + 4 * n4;
  }
  for (int64_t e = e_tail + threadIdx.x; e < e1; e += blockDim.x) {
    float w = sg.w[e], g = sg.g[e];
    float* p0 = sg.s0 ? sg.s0 + e : &dummy0;
    float* p1 = sg.s1 ? sg.s1 + e : &dummy1;
    apply_rule(r, w, g, p0, p1);
    sg.w[e] = w;
    sg.g[e] = g;
  }
}

__global__ void update_rows_kernel(RuleArgs r, float* w, float* g, float* s0, float* s1, int dim,
                                   const int64_t* __restrict__ ids, int n_rows) {
  pdl_prologue();
  const int64_t total = (int64_t)n_rows * dim;
  float dummy0 = 0.f, dummy1 = 0.f;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = t / dim, c = t - u * dim;
    const int64_t e = ids[u] * dim + c;
    float wv = w[e], gv = g[e];
    apply_rule(r, wv, gv, s0 ? s0 + e : &dummy0, s1 ? s1 + e : &dummy1);
    w[e] = wv;
    g[e] = gv;
  }
}

__global__ void scale_kernel(float* y, int64_t n, float alpha) {
  pdl_prologue();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    y[t] *= alpha;
}
__global__ void fill_kernel(float* y, int64_t n, float v) {
  pdl_prologue();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    y[t] = v;
}

inline int grid_for(int64_t n) {
  const int64_t cap = 148 * 32;
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b > cap) b = cap;
  return b < 1 ? 1 : static_cast<int>(b);
}

}  // namespace

// ------------------------------------------------------------------ launchers

int launch_ew_fwd(const EwArgs& a, cudaStream_t s) {
  const int64_t total = (int64_t)a.elem * a.batch * a.n;
  if (total == 0) return 0;
  launch_k(ew_fwd_kernel, grid_for(total), kThreads, 0, s, a);
  return 1;
}

int launch_ew_bwd(const EwArgs& a, cudaStream_t s) {
  const bool bcast_ok = a.kind == EW_ADD || a.kind == EW_CMULT || a.kind == EW_SCALE;
  if (bcast_ok && (a.a_b1 || a.b_b1) && a.batch > 1) {
    launch_k(ew_bwd_bcast_kernel, grid_for((int64_t)a.elem * a.n), kThreads, 0, s, a);
  } else {
    EwArgs c = a;
    c.a_b1 = c.b_b1 = 0;
    launch_k(ew_bwd_flat_kernel, grid_for((int64_t)a.elem * a.batch * a.n), kThreads, 0, s, c);
  }
  return 1;
}

int launch_chain_fwd(const ChainArgs& a, cudaStream_t s) {
  if ((int64_t)a.size * a.n < 2048 && a.len >= 8) {
    launch_k(chain_fwd_seq_kernel, a.size * a.n, 256, 0, s, a);
    return 1;
  }
  launch_k(chain_fwd_kernel, grid_for((int64_t)a.size * a.n), kThreads, 0, s, a);
  return 1;
}
int launch_chain_bwd(const ChainArgs& a, cudaStream_t s) {
  if (a.distinct) {
    launch_k(chain_bwd_par_kernel, grid_for((int64_t)(2 * a.len) * a.n * a.size), kThreads, 0, s, a);
    return 1;
  }
  launch_k(chain_bwd_kernel, grid_for((int64_t)a.size * a.n), kThreads, 0, s, a);
  return 1;
}

int launch_cell_fwd(const CellArgs& a, cudaStream_t s) {
  const int g = a.n * (int)(((int64_t)a.batch * a.H + 255) / 256);
  switch (a.m) {
    case 0: launch_k(cell_fwd_kernel<0>, g, kThreads, 0, s, a); break;
    case 1: launch_k(cell_fwd_kernel<1>, g, kThreads, 0, s, a); break;
    default: launch_k(cell_fwd_kernel<2>, g, kThreads, 0, s, a); break;
  }
  return 1;
}

int launch_cell_bwd(const CellArgs& a, cudaStream_t s) {
  bool bcast = false;
  for (int k = 0; k < a.m; ++k) bcast = bcast || (a.cext_b1[k] && a.batch > 1);
  // broadcast variant: exactly one block per (cell, 32-unit chunk), single pass
  const int g = bcast ? a.n * ((a.H + 31) / 32) : a.n * (int)(((int64_t)a.batch * a.H + 255) / 256);
  switch (a.m * 2 + (bcast ? 1 : 0)) {
    case 0: launch_k(cell_bwd_kernel<0, false>, g, kThreads, 0, s, a); break;
    case 1: launch_k(cell_bwd_kernel<0, true>, g, kThreads, 0, s, a); break;
    case 2: launch_k(cell_bwd_kernel<1, false>, g, kThreads, 0, s, a); break;
    case 3: launch_k(cell_bwd_kernel<1, true>, g, kThreads, 0, s, a); break;
    case 4: launch_k(cell_bwd_kernel<2, false>, g, kThreads, 0, s, a); break;
    default: launch_k(cell_bwd_kernel<2, true>, g, kThreads, 0, s, a); break;
  }
  return 1;
}

int launch_pnls2_fwd(const Pnls2Args& a, cudaStream_t s) {
  if (a.n <= 0) return 0;
  launch_k(pnls2_fwd_kernel, a.n, kThreads, 0, s, a);
  return 1;
}

int launch_pnls2_bwd(const Pnls2Args& a, cudaStream_t s) {
  if (a.n <= 0) return 0;
  launch_k(pnls2_bwd_kernel, a.n, kThreads, 0, s, a);
  return 1;
}

int launch_gru_fwd(const GruArgs& a, bool part_b, cudaStream_t s) {
  const int64_t total = (int64_t)a.n * a.batch * a.H;
  if (part_b) launch_k(gru_fwd_kernel<true>, grid_for(total), kThreads, 0, s, a);
  else launch_k(gru_fwd_kernel<false>, grid_for(total), kThreads, 0, s, a);
  return 1;
}

int launch_gru_bwd(const GruArgs& a, bool part_b, cudaStream_t s) {
  const int64_t total = (int64_t)a.n * a.H;
  if (part_b) launch_k(gru_bwd_kernel<true>, grid_for(total), kThreads, 0, s, a);
  else launch_k(gru_bwd_kernel<false>, grid_for(total), kThreads, 0, s, a);
  return 1;
}

int launch_pick_fwd(const PickArgs& a, cudaStream_t s) {
  launch_k(pick_fwd_kernel, grid_for((int64_t)a.n * a.batch * a.width), kThreads, 0, s, a);
  return 1;
}
int launch_pick_bwd(const PickArgs& a, cudaStream_t s) {
  launch_k(pick_bwd_kernel, grid_for((int64_t)a.n * a.batch * a.width), kThreads, 0, s, a);
  return 1;
}
int launch_concat_fwd(const ConcatArgs& a, cudaStream_t s) {
  launch_k(concat_fwd_kernel, grid_for((int64_t)a.n * a.batch * a.total), kThreads, 0, s, a);
  return 1;
}
int launch_concat_bwd(const ConcatArgs& a, cudaStream_t s) {
  launch_k(concat_bwd_kernel, grid_for((int64_t)a.n * a.batch * a.total), kThreads, 0, s, a);
  return 1;
}
int launch_sum_batches_fwd(const SumBatchesArgs& a, cudaStream_t s) {
  launch_k(sum_batches_fwd_kernel, grid_for((int64_t)a.n * a.elem), kThreads, 0, s, a);
  return 1;
}
int launch_sum_batches_bwd(const SumBatchesArgs& a, cudaStream_t s) {
  launch_k(sum_batches_bwd_kernel, grid_for((int64_t)a.n * a.batch * a.elem), kThreads, 0, s, a);
  return 1;
}

int launch_softmax_fwd(const RowArgs& a, cudaStream_t s) { return launch_rows<0>(a, s); }
int launch_softmax_bwd(const RowArgs& a, cudaStream_t s) { return launch_rows<1>(a, s); }
int launch_pnls_fwd(const RowArgs& a, cudaStream_t s) { return launch_rows<2>(a, s); }
int launch_pnls_bwd(const RowArgs& a, cudaStream_t s) { return launch_rows<3>(a, s); }

int launch_gather_rows(const float* table, int dim, const int64_t* ids, float* const* out_rows, int rows,
                       cudaStream_t s) {
  if (rows <= 0) return 0;
  launch_k(gather_rows_kernel, (rows + 7) / 8, 256, 0, s, table, dim, ids, out_rows, rows);
  return 1;
}

int plan_scatter_items(const int* seg, int n_unique, std::vector<ScatterItem>& items, int* n_partials,
                       int* n_long) {
  items.clear();
  int pb = 0, nl = 0;
  for (int u = 0; u < n_unique; ++u) {
    const int k0 = seg[u], k1 = seg[u + 1], len = k1 - k0;
    if (len <= kScatterChunk) {
      items.push_back(ScatterItem{u, k0, k1, 0, 0, 0, 0, 0});
      continue;
    }
    const int nc = (len + kScatterChunk - 1) / kScatterChunk;
    for (int c = 0; c < nc; ++c)
      items.push_back(ScatterItem{u, k0 + c * kScatterChunk, std::min(k1, k0 + (c + 1) * kScatterChunk), c, nc, pb, nl,
                                  0});
    pb += nc;
    ++nl;
  }
  *n_partials = pb;
  *n_long = nl;
  return (int)items.size();
}

int launch_scatter_rows(float* table_grad, int dim, const int64_t* uniq_ids, const ScatterItem* items, int n_items,
                        const float* const* src_rows, float* partials, int* counters, float scale, bool set_mean,
                        cudaStream_t s) {
  if (n_items <= 0) return 0;
  const int grid = (n_items + 7) / 8;
  if (set_mean)
    launch_k(scatter_rows_kernel<true>, grid, 256, 0, s, table_grad, dim, uniq_ids, items, n_items, src_rows, partials,
             counters, scale);
  else
    launch_k(scatter_rows_kernel<false>, grid, 256, 0, s, table_grad, dim, uniq_ids, items, n_items, src_rows,
             partials, counters, scale);
  return 1;
}

int launch_pack_rows(const float* table, int dim, const int64_t* ids, float* out, int n, cudaStream_t s) {
  if (n <= 0) return 0;
  launch_k(pack_rows_kernel, grid_for((int64_t)n * dim), kThreads, 0, s, table, dim, ids, out, n);
  return 1;
}

int launch_matmul_fwd(const MatmulArgs& a, cudaStream_t s) {
  launch_k(matmul_fwd_kernel, grid_for((int64_t)a.n * a.batch * a.m * a.p), kThreads, 0, s, a);
  return 1;
}
int launch_matmul_bwd(const MatmulArgs& a, cudaStream_t s) {
  launch_k(matmul_bwd_a_kernel, grid_for((int64_t)a.n * a.batch * a.m * a.k), kThreads, 0, s, a);
  launch_k(matmul_bwd_x_kernel, grid_for((int64_t)a.n * a.batch * a.k * a.p), kThreads, 0, s, a);
  return 2;
}

int launch_affine_generic_fwd(const AffineGenericArgs& a, cudaStream_t s) {
  launch_k(affine_generic_fwd_kernel, grid_for((int64_t)a.n * a.batch * a.m), kThreads, 0, s, a);
  return 1;
}
int launch_affine_generic_bwd(const AffineGenericArgs& a, cudaStream_t s) {
  int launches = 0;
  launch_k(affine_generic_bwd_kernel, grid_for((int64_t)a.n * a.batch * a.m), kThreads, 0, s, a, 0, 0);
  ++launches;
  for (int k = 0; k < a.terms; ++k) {
    launch_k(affine_generic_bwd_kernel, grid_for((int64_t)a.n * a.batch * a.m * a.kdim[k]), kThreads, 0, s, a, 1, k);
    launch_k(affine_generic_bwd_kernel, grid_for((int64_t)a.n * a.batch * a.kdim[k]), kThreads, 0, s, a, 2, k);
    launches += 2;
  }
  return launches;
}

int launch_colsum_group(ColsumGroup G, float* work, int64_t work_floats, cudaStream_t s) {
  if (G.n <= 0) return 0;
  // jobs with 16 B rows (width % 4 == 0): grouped row-segment partials, then
  // one final pass; the others below
  int launched = 0;
  {
    ColsumGroup W{}, N{};
    W.nowait = G.nowait;
    int64_t off = 0;
    int pb = 0, fb = 0;
    for (int q = 0; q < G.n; ++q) {
      ColsumJob J = G.j[q];
      const int chunks = (J.n_rows + kColsumWideRows - 1) / kColsumWideRows;
      const bool wide = J.vec && J.width % 4 == 0 && J.width >= 64 && off + (int64_t)chunks * J.width <= work_floats;
      if (!wide) {
        N.j[N.n++] = J;
        continue;
      }
      J.chunks = chunks;
      J.work = work + off;
      off += ((int64_t)chunks * J.width + 63) & ~int64_t(63);
      J.pb0 = pb;
      J.fb0 = fb;
      pb += chunks * ((J.width / 4 + 511) / 512);
      fb += (J.width + 31) / 32;
      W.j[W.n++] = J;
    }
    if (W.n) {
      launch_k(colsum_wide_partial_kernel, pb, 256, 0, s, W);
      launch_k(colsum_final_group_kernel, fb, 256, 0, s, W);
      launched = 2;
    }
    if (N.n == 0) return launched;
    G = N;
    work += off;
    work_floats -= off;
  }
  // chunking per job as launch_colsum_rows, partials packed into the scratch
  int pb = 0, fb = 0;
  int64_t off = 0;
  for (int q = 0; q < G.n; ++q) {
    ColsumJob& J = G.j[q];
    const int xb = (J.width + 255) / 256;
    int chunks = (2 * 148 * 8 + xb - 1) / xb;
    chunks = std::min(chunks, std::max(1, J.n_rows / 8));
    const int64_t left = work_floats - off;
    chunks = (int)std::min<int64_t>(chunks, std::max<int64_t>(1, left / std::max(1, J.width)));
    chunks = std::min(chunks, 1024);
    if ((int64_t)chunks * J.width > left) return -1;
    J.chunks = chunks;
    J.work = work + off;
    off += ((int64_t)chunks * J.width + 63) & ~int64_t(63);
    J.pb0 = pb;
    J.fb0 = fb;
    pb += xb * chunks;
    fb += (J.width + 31) / 32;
  }
  launch_k(colsum_partial_group_kernel, pb, 256, 0, s, G);
  launch_k(colsum_final_group_kernel, fb, 256, 0, s, G);
  return launched + 2;
}

int launch_colsum_rows(float* dst, const float* const* rows, int n_rows, int width, float* work, int64_t work_floats,
                       cudaStream_t s) {
  if (n_rows <= 0) return 0;
  // enough (column block, row chunk) blocks to fill the device twice over,
  // chunks of >= 8 rows, partials bounded by the scratch
  const int xb = (width + 255) / 256;
  int chunks = (2 * 148 * 8 + xb - 1) / xb;
  chunks = std::min(chunks, std::max(1, n_rows / 8));
  chunks = (int)std::min<int64_t>(chunks, std::max<int64_t>(1, work_floats / std::max(1, width)));
  chunks = std::min(chunks, 1024);
  dim3 g1((width + 255) / 256, chunks);
  launch_k(colsum_partial_kernel, g1, 256, 0, s, rows, n_rows, width, chunks, work);
  launch_k(colsum_final_kernel, (width + 31) / 32, 256, 0, s, dst, work, width, chunks);
  return 2;
}

int launch_row_reduce_scatter(float* const* dst_rows, const int* seg, const float* src, int n_targets, int width,
                              cudaStream_t s) {
  if (n_targets <= 0) return 0;
  launch_k(row_reduce_scatter_kernel, n_targets, 256, 0, s, dst_rows, seg, src, n_targets, width);
  return 1;
}

int launch_update_dense(const RuleArgs& r, const TensorSeg* segs_dev, int nseg, int64_t total_blocks, cudaStream_t s) {
  if (nseg <= 0 || total_blocks <= 0) return 0;
  launch_k(update_dense_kernel, static_cast<unsigned>(total_blocks), 256, 0, s, r, segs_dev, nseg);
  return 1;
}

int launch_update_rows(const RuleArgs& r, float* w, float* g, float* s0, float* s1, int dim, const int64_t* ids,
                       int n_rows, cudaStream_t s) {
  if (n_rows <= 0) return 0;
  launch_k(update_rows_kernel, grid_for((int64_t)n_rows * dim), kThreads, 0, s, r, w, g, s0, s1, dim, ids, n_rows);
  return 1;
}

int launch_scale(float* y, int64_t n, float alpha, cudaStream_t s) {
  if (n <= 0) return 0;
  launch_k(scale_kernel, grid_for(n), kThreads, 0, s, y, n, alpha);
  return 1;
}
int launch_fill(float* y, int64_t n, float v, cudaStream_t s) {
  if (n <= 0) return 0;
  launch_k(fill_kernel, grid_for(n), kThreads, 0, s, y, n, v);
  return 1;
}

int update_chunk() { return kUpdChunk; }

}  // namespace dg
