// Standalone timing of the grouped GEMM on the RNNLM shapes (CUDA events,
// hot L2, 50 reps).  Build: see tools/build_tools.sh.  Diagnostic only.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
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

int main() {
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
