// Standalone timing of the grouped GEMM on the RNNLM shapes (CUDA events,
// hot L2, 50 reps).  Build: see tools/build_tools.sh.  Diagnostic only.
#include <cuda_runtime.h>

#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "../paper_1701_03980_b200/csrc/kernels.cuh"

using namespace dg;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

struct Shape {
  int M, N, K;
};

static float* dalloc(size_t n) {
  float* p;
  CK(cudaMalloc(&p, n * 4));
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)((i * 2654435761u) % 1000) / 1000.f - 0.5f;
  CK(cudaMemcpy(p, h.data(), n * 4, cudaMemcpyHostToDevice));
  return p;
}

// one launch over `shapes` (a_kmajor / b_nmajor as given); returns us per launch
static double run(const char* name, std::vector<Shape> shapes, bool ak, bool bn, bool tables, float* work,
                  int* counters, void* dprobs, int force_split) {
  std::vector<GemmProblem> probs;
  std::vector<float*> bufs;
  for (auto& s : shapes) {
    GemmProblem p{};
    p.M = s.M;
    p.N = s.N;
    p.n_seg = 1;
    p.seg[0].K = s.K;
    float* A = dalloc((size_t)s.M * s.K);
    float* B = dalloc((size_t)s.K * s.N);
    float* C = dalloc((size_t)s.M * s.N);
    bufs.push_back(A);
    bufs.push_back(B);
    bufs.push_back(C);
    p.seg[0].A.base = A;
    p.seg[0].A.ld = ak ? s.M : s.K;
    p.seg[0].B.base = B;
    p.seg[0].B.ld = bn ? s.K : s.N;
    p.C.base = C;
    p.C.ld = s.N;
    if (tables) {
      const int ra = ak ? s.K : s.M;
      std::vector<const float*> rows(ra);
      for (int i = 0; i < ra; ++i) rows[i] = A + (size_t)i * p.seg[0].A.ld;
      const float** d;
      CK(cudaMalloc(&d, ra * sizeof(void*)));
      CK(cudaMemcpy(d, rows.data(), ra * sizeof(void*), cudaMemcpyHostToDevice));
      p.seg[0].A.rows = d;
      p.seg[0].A.rows_aligned = 1;
    }
    p.accumulate = 1;
    probs.push_back(p);
  }
  GemmLaunch L = gemm_plan(probs, ak, bn, 64ll << 20, 1 << 18);
  if (force_split > 0) {
    // re-plan with a forced split count
    int64_t cta = 0, woff = 0, ctr = 0;
    for (auto& p : probs) {
      p.splits = force_split;
      p.cta0 = (int)cta;
      p.counter0 = (int)ctr;
      p.work_off = woff;
      cta += (int64_t)p.tiles * force_split;
      ctr += p.tiles;
      woff += (int64_t)force_split * p.tiles * 128 * 128;
      L.cluster = L.cfg != 0 && force_split > 1 ? force_split : 0;
    }
    L.ctas = (int)cta;
  }
  CK(cudaMemcpy(dprobs, probs.data(), probs.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 5; ++i) launch_gemm_group(L, (const GemmProblem*)dprobs, work, counters, 0);
  CK(cudaEventRecord(e0));
  const int reps = 50;
  for (int i = 0; i < reps; ++i) launch_gemm_group(L, (const GemmProblem*)dprobs, work, counters, 0);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  double us = 1e3 * ms / reps;
  double fl = L.flops;
  printf("%-34s cfg %d ctas %5d splits %2d  %8.2f us  %7.2f TFLOP/s\n", name, L.cfg, L.ctas, probs[0].splits, us,
         fl / (us * 1e-6) / 1e12);
  for (float* b : bufs) cudaFree(b);
  return us;
}

__global__ void empty_kernel() {}
__global__ void copy_kernel(const float* a, float* b, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i] * 2.f;
}

static void floor_timings() {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float* a = dalloc(1 << 16);
  float* b = dalloc(1 << 16);
  for (int variant = 0; variant < 3; ++variant) {
    for (int i = 0; i < 10; ++i) empty_kernel<<<1, 32>>>();
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 200; ++i) {
      if (variant == 0) empty_kernel<<<1, 32>>>();
      else if (variant == 1) empty_kernel<<<148 * 4, 128>>>();
      else copy_kernel<<<64, 256>>>(a, b, 1 << 14);
    }
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("floor %-28s %6.2f us/launch\n",
           variant == 0 ? "empty <<<1,32>>>" : (variant == 1 ? "empty <<<592,128>>>" : "copy 16k floats"),
           1e3 * ms / 200);
  }
}

static int g_force_cluster = 0;
static int g_chunk = 0;
static bool g_simt = false;

// correctness: tensor-core path vs an fp64 host reference (sampled rows)
static void check_tc(const char* name, int M, int N, int K, bool ak, bool bn, bool tables, void* dprobs) {
  std::vector<float> hA((size_t)M * K), hB((size_t)K * N);
  for (size_t i = 0; i < hA.size(); ++i) hA[i] = (float)(((i * 2654435761u) >> 7) % 2001) / 1000.f - 1.f;
  for (size_t i = 0; i < hB.size(); ++i) hB[i] = (float)(((i * 40503u + 7) >> 3) % 1999) / 1000.f - 1.f;
  // A(m,k): ak ? A[k*M + m] : A[m*K + k];  B(k,n): bn ? B[n*K + k] : B[k*N + n]
  float *A, *B, *C;
  CK(cudaMalloc(&A, hA.size() * 4));
  CK(cudaMalloc(&B, hB.size() * 4));
  CK(cudaMalloc(&C, (size_t)M * N * 4));
  CK(cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(C, 0, (size_t)M * N * 4));
  GemmProblem p{};
  p.M = M;
  p.N = N;
  p.n_seg = 1;
  p.seg[0].K = K;
  p.seg[0].A.base = A;
  p.seg[0].A.ld = ak ? M : K;
  p.seg[0].B.base = B;
  p.seg[0].B.ld = bn ? K : N;
  p.C.base = C;
  p.C.ld = N;
  if (tables) {
    const int ra = ak ? K : M;
    std::vector<const float*> rows(ra);
    for (int i = 0; i < ra; ++i) rows[i] = A + (size_t)i * p.seg[0].A.ld;
    const float** d;
    CK(cudaMalloc(&d, ra * sizeof(void*)));
    CK(cudaMemcpy(d, rows.data(), ra * sizeof(void*), cudaMemcpyHostToDevice));
    p.seg[0].A.rows = d;
    p.seg[0].A.rows_aligned = 1;
  }
  std::vector<GemmProblem> probs{p};
  GemmLaunch L = tc_gemm_plan(probs, ak, bn);
  if (g_chunk > 0) L.chunk = g_chunk;
  if (g_force_cluster > 0) {  // forced split-K (cluster size) for accuracy studies
    int64_t cta = 0;
    for (auto& q : probs) {
      q.splits = g_force_cluster;
      q.cta0 = (int)cta;
      cta += (int64_t)q.tiles * g_force_cluster;
    }
    L.cluster = g_force_cluster;
    L.ctas = (int)cta;
  }
  if (g_simt) {
    static float* work = nullptr;
    static int* counters = nullptr;
    if (!work) {
      CK(cudaMalloc(&work, 64 << 20));
      CK(cudaMalloc(&counters, 1 << 20));
      CK(cudaMemset(counters, 0, 1 << 20));
    }
    L = gemm_plan(probs, ak, bn, 16 << 20, 1 << 18);
    CK(cudaMemcpy(dprobs, probs.data(), sizeof(GemmProblem), cudaMemcpyHostToDevice));
    launch_gemm_group(L, (const GemmProblem*)dprobs, work, counters, 0);
  } else {
    CK(cudaMemcpy(dprobs, probs.data(), sizeof(GemmProblem), cudaMemcpyHostToDevice));
    launch_tc_gemm(L, (const GemmProblem*)dprobs, 0);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> hC((size_t)M * N);
  CK(cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0, scale = 0;
  for (int m = 0; m < M; m += std::max(1, M / 37)) {
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) {
        const double a = ak ? hA[(size_t)k * M + m] : hA[(size_t)m * K + k];
        const double b = bn ? hB[(size_t)n * K + k] : hB[(size_t)k * N + n];
        s += a * b;
      }
      worst = std::max(worst, std::fabs(s - hC[(size_t)m * N + n]));
      scale = std::max(scale, std::fabs(s));
    }
  }
  printf("check %-30s M%5d N%5d K%5d cluster %d  max|err| %.3e  (scale %.3e, rel %.2e) %s\n", name, M, N, K,
         L.cluster, worst, scale, worst / scale, worst / scale < 1e-5 ? "OK" : "FAIL");
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
}

static int g_chunk_dummy = 0;
static double run_tc(const char* name, std::vector<Shape> shapes, bool ak, bool bn, void* dprobs) {
  std::vector<GemmProblem> probs;
  std::vector<float*> bufs;
  for (auto& s : shapes) {
    GemmProblem p{};
    p.M = s.M;
    p.N = s.N;
    p.n_seg = 1;
    p.seg[0].K = s.K;
    float* A = dalloc((size_t)s.M * s.K);
    float* B = dalloc((size_t)s.K * s.N);
    float* C = dalloc((size_t)s.M * s.N);
    bufs.push_back(A);
    bufs.push_back(B);
    bufs.push_back(C);
    p.seg[0].A.base = A;
    p.seg[0].A.ld = ak ? s.M : s.K;
    p.seg[0].B.base = B;
    p.seg[0].B.ld = bn ? s.K : s.N;
    p.C.base = C;
    p.C.ld = s.N;
    p.accumulate = 1;
    probs.push_back(p);
  }
  GemmLaunch L = tc_gemm_plan(probs, ak, bn);
  if (g_chunk > 0) L.chunk = g_chunk;
  CK(cudaMemcpy(dprobs, probs.data(), probs.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) launch_tc_gemm(L, (const GemmProblem*)dprobs, 0);
  CK(cudaEventRecord(e0));
  const int reps = 20;
  for (int i = 0; i < reps; ++i) launch_tc_gemm(L, (const GemmProblem*)dprobs, 0);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double us = 1e3 * ms / reps;
  printf("TC  %-30s ctas %5d cluster %d  %8.2f us  %7.2f TFLOP/s (3xTF32: %.1f TF/s issued)\n", name, L.ctas,
         L.cluster, us, L.flops / (us * 1e-6) / 1e12, 3 * L.flops / (us * 1e-6) / 1e12);
  for (float* b : bufs) cudaFree(b);
  return us;
}

int main() {
  floor_timings();
  {
    void* dp;
    CK(cudaMalloc(&dp, 1 << 16));
    check_tc("rowmajor A, n-major B", 256, 256, 96, false, true, false, dp);
    check_tc("rowmajor A, k-major B", 256, 384, 128, false, false, false, dp);
    check_tc("k-major A, k-major B", 256, 256, 160, true, false, false, dp);
    check_tc("k-major A, n-major B", 384, 256, 64, true, true, false, dp);
    check_tc("ragged + tables", 300, 200, 100, false, false, true, dp);
    check_tc("split-K cluster", 128, 128, 4096, false, true, false, dp);
    // accuracy vs accumulation-chain length: the aggregated LSTM dW shape
    for (int s : {1, 2, 4, 8}) {
      g_force_cluster = s;
      check_tc("dW-like k-major A, cluster", 256, 1024, 2176, true, false, false, dp);
    }
    g_force_cluster = 0;
    for (int ch : {1, 2, 4, 1000}) {
      g_chunk = ch;
      check_tc("dW-like, TMEM drain every (ch)", 256, 1024, 2176, true, false, false, dp);
      check_tc("dX-like, TMEM drain every (ch)", 256, 256, 10000, false, true, false, dp);
      run_tc("  dX 2176x256x10000", {{2176, 256, 10000}}, false, true, dp);
      run_tc("  fwd 2176x10000x256", {{2176, 10000, 256}}, false, false, dp);
    }
    g_chunk = 0;
    g_simt = true;
    check_tc("dW-like SIMT (blocked sum)", 256, 1024, 2176, true, false, false, dp);
    check_tc("dX-like SIMT (blocked sum)", 256, 256, 10000, false, true, false, dp);
    g_simt = false;
    check_tc("dX-like TC", 256, 256, 10000, false, true, false, dp);
    run_tc("fwd 2176x10000x256", {{2176, 10000, 256}}, false, false, dp);
    run_tc("dX 2176x256x10000", {{2176, 256, 10000}}, false, true, dp);
    run_tc("dW 256x10000x2176", {{256, 10000, 2176}}, true, false, dp);
    run_tc("dW LSTM 384x1024x2176", {{384, 1024, 2176}}, true, false, dp);
  }
  float* work;
  int* counters;
  void* dprobs;
  CK(cudaMalloc(&work, 256ll << 20));
  CK(cudaMalloc(&counters, 1 << 20));
  CK(cudaMemset(counters, 0, 1 << 20));
  CK(cudaMalloc(&dprobs, 1 << 16));
  // empty kernel launch latency reference
  printf("-- recurrent level, forward (2 problems, W^T k-major)\n");
  run("fwd L0+L1 64x1024x{384,512}", {{64, 1024, 384}, {64, 1024, 512}}, false, false, true, work, counters, dprobs, 0);
  for (int s : {1, 2, 4, 8})
    run("  forced split", {{64, 1024, 384}, {64, 1024, 512}}, false, false, true, work, counters, dprobs, s);
  printf("-- recurrent level, dX (n-major W)\n");
  run("dX 64x256x1024 + 64x128x1024", {{64, 256, 1024}, {64, 128, 1024}}, false, true, true, work, counters, dprobs,
      0);
  for (int s : {1, 2, 4, 8})
    run("  forced split", {{64, 256, 1024}, {64, 128, 1024}}, false, true, true, work, counters, dprobs, s);
  printf("-- output layer\n");
  run("fwd 2176x10000x256", {{2176, 10000, 256}}, false, false, true, work, counters, dprobs, 0);
  run("dX 2176x256x10000", {{2176, 256, 10000}}, false, true, true, work, counters, dprobs, 0);
  run("dW 256x10000x2176 (k-major A)", {{256, 10000, 2176}}, true, false, false, work, counters, dprobs, 0);
  run("dW LSTM 384x1024x2176", {{384, 1024, 2176}}, true, false, false, work, counters, dprobs, 0);
  return 0;
}
