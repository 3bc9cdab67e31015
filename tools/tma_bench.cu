// Correctness + timing of the TMA 3xTF32 GEMM (tmagemm.cu) against an fp64
// host reference, on the output-layer shapes of the PTB RNNLM.  Diagnostic
// only; build: tools/build_tools.sh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

static float* dfill(std::vector<float>& h, size_t n, unsigned seed) {
  h.resize(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)(((i + seed) * 2654435761u) % 2001) / 1000.f - 1.0f;
  float* p;
  CK(cudaMalloc(&p, n * 4));
  CK(cudaMemcpy(p, h.data(), n * 4, cudaMemcpyHostToDevice));
  return p;
}

// a_mn: A stored K x M (row k holds M values), else M x K; b_mn: B stored K x N, else N x K
static void run(const char* name, int M, int N, int K, bool a_mn, bool b_mn, bool check, int reps) {
  std::vector<float> hA, hB, hC;
  float* A = dfill(hA, (size_t)M * K, 1);
  float* B = dfill(hB, (size_t)K * N, 7);
  float* C = dfill(hC, (size_t)M * N, 13);
  float *Alo, *Blo;
  CK(cudaMalloc(&Alo, tma_lo_floats(a_mn ? K : M, a_mn ? M : K) * 4));
  CK(cudaMalloc(&Blo, tma_lo_floats(b_mn ? K : N, b_mn ? N : K) * 4));
  TmaOperands o{};
  o.M = M;
  o.N = N;
  o.K = K;
  o.a_mn = a_mn;
  o.b_mn = b_mn;
  o.A = A;
  o.lda = a_mn ? M : K;
  o.B = B;
  o.ldb = b_mn ? N : K;
  o.A_lo = Alo;
  o.B_lo = Blo;
  o.C.base = C;
  o.C.ld = N;
  static float* ws = nullptr;
  static int* cnt = nullptr;
  const int64_t ws_floats = (int64_t)64 << 20;
  if (!ws) {
    CK(cudaMalloc(&ws, ws_floats * 4));
    CK(cudaMalloc(&cnt, 65536 * 4));
    CK(cudaMemset(cnt, 0, 65536 * 4));
  }
  if (!getenv("TMA_NO_WS")) {
    o.ws = ws;
    o.ws_floats = ws_floats;
    o.cnt = cnt;
    o.cnt_cap = 65536;
  }
  o.accumulate = 1;
  std::vector<float> hb;
  float* bias = nullptr;
  const bool fwd_like = name[0] == 'f';  // logits = H W^T + b (overwrite, broadcast bias row)
  if (fwd_like) {
    bias = dfill(hb, (size_t)N, 29);
    o.bias.base = bias;
    o.bias.ld = 0;
    o.accumulate = 0;
  }
  TmaGemmPlan p;
  if (!tma_gemm_make(o, &p)) {
    printf("%s: tensor map creation failed\n", name);
    exit(1);
  }
  if (launch_tma_gemm(p, true, true, 0) < 0) {
    printf("%s: launch failed: %s\n", name, cudaGetErrorString(cudaGetLastError()));
    exit(1);
  }
  CK(cudaDeviceSynchronize());
  if (check) {
    std::vector<float> out((size_t)M * N);
    CK(cudaMemcpy(out.data(), C, out.size() * 4, cudaMemcpyDeviceToHost));
    double worst = 0, scale = 0;
    for (int m = 0; m < M; m += std::max(1, M / 41)) {
      for (int n = 0; n < N; n += std::max(1, N / 97)) {
        double s = fwd_like ? hb[n] : hC[(size_t)m * N + n];
        for (int k = 0; k < K; ++k) {
          const double a = a_mn ? hA[(size_t)k * M + m] : hA[(size_t)m * K + k];
          const double b = b_mn ? hB[(size_t)k * N + n] : hB[(size_t)n * K + k];
          s += a * b;
        }
        worst = std::max(worst, std::fabs(s - out[(size_t)m * N + n]));
        scale = std::max(scale, std::fabs(s));
      }
    }
    printf("check %-26s M%5d N%5d K%5d a_mn %d b_mn %d split %d%s  max|err| %.3e (scale %.3e, rel %.2e) %s\n", name, M,
           N, K, a_mn, b_mn, p.args.splits, p.args.gsplit ? "g" : "c", worst, scale, worst / scale, worst / scale < 8e-6 ? "OK" : "FAIL");
  }
  if (getenv("TMA_PROF")) {  // DG_TMA_DBG bit 10: CTA 0 wait timeline of one launch
    CK(cudaDeviceSynchronize());
    launch_tma_gemm(p, false, false, 0);
    CK(cudaDeviceSynchronize());
    static long long t[6][256][2];
    tma_prof_read(&t[0][0][0]);
    long long base = t[2][0][0];
    const char* role[6] = {"prod empty", "mma acc_empty", "mma conv", "conv full", "epi acc_full", "epi end(pers)"};
    printf("prof %s (cycles rel. to first MMA wait; wait duration)\n", name);
    for (int r = 0; r < 6; ++r) {
      printf("  %-14s", role[r]);
      int shown = 0;
      for (int j = 0; j < 256 && shown < 40; ++j) {
        if (t[r][j][0] == 0 && t[r][j][1] == 0) continue;
        printf(" [%d]%lld+%lld", j, t[r][j][0] - base, t[r][j][1] - t[r][j][0]);
        ++shown;
      }
      printf("\n");
    }
    if (getenv("TMA_PROF_EPI")) {
      for (int i = 1; i <= 3; ++i) {
        printf("  epi tile %d chunks (ld, staged, bar, stored):", i);
        for (int h = 0; h < 4; ++h)
          printf(" [%lld %lld %lld %lld]", t[4][64 + i * 16 + h * 4][0] - base, t[4][64 + i * 16 + h * 4 + 1][0] - base,
                 t[4][64 + i * 16 + h * 4 + 2][0] - base, t[4][64 + i * 16 + h * 4 + 3][0] - base);
        printf("\n");
      }
    }
    printf("  phases (clk from kernel start): mainloop end %lld, part stored %lld, sync %lld, cluster sync %lld, end %lld\n",
           t[5][1][0] - t[5][0][0], t[5][2][0] - t[5][0][0], t[5][3][0] - t[5][0][0], t[5][4][0] - t[5][0][0],
           t[5][5][0] - t[5][0][0]);
    memset(t, 0, sizeof t);
  }
  if (reps > 0) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) launch_tma_gemm(p, false, false, 0);
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) launch_tma_gemm(p, false, false, 0);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = 1e3 * ms / reps;
    printf("time  %-26s ctas %5d split %d%s  %8.2f us  %7.2f TFLOP/s (3xTF32 issued %.1f TF/s)\n", name, p.ctas,
           p.args.splits, p.args.gsplit ? "g" : "c", us, p.flops / (us * 1e-6) / 1e12, 3 * p.flops / (us * 1e-6) / 1e12);
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) launch_tma_gemm(p, true, true, 0);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("      %-26s with lo splits %8.2f us\n", name, 1e3 * ms / reps);
  }
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  cudaFree(Alo);
  cudaFree(Blo);
  if (bias) cudaFree(bias);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // timing only (diagnostic variants via DG_TMA_DBG / DG_TMA_CONV)
    run("fwd 2176x10000x256", 2176, 10000, 256, false, true, false, 20);
    run("dX 2176x256x10000", 2176, 256, 10000, false, false, false, 20);
    run("dW 256x10000x2176", 256, 10000, 2176, true, true, false, 20);
    run("dW LSTM 512x1024x2240", 512, 1024, 2240, true, true, false, 20);
    run("fwd 2752x10000x256", 2752, 10000, 256, false, true, false, 20);
    run("Gx 2752x1024x256", 2752, 1024, 256, false, true, false, 20);
    return 0;
  }
  run("kmajor/kmajor", 256, 256, 96, false, false, true, 0);
  run("kmajor A / mn B", 256, 384, 128, false, true, true, 0);
  run("mn A / kmajor B", 256, 256, 160, true, false, true, 0);
  run("mn A / mn B", 384, 256, 64, true, true, true, 0);
  run("ragged", 300, 200, 100, false, true, true, 0);
  run("ragged mn", 300, 200, 100, true, true, true, 0);
  run("split-K", 128, 128, 4096, false, false, true, 0);
  run("dX-like K=10000", 256, 256, 10000, false, false, true, 0);
  run("fwd 2176x10000x256", 2176, 10000, 256, false, true, true, 20);
  run("dX 2176x256x10000", 2176, 256, 10000, false, false, true, 20);
  run("dW 256x10000x2176", 256, 10000, 2176, true, true, true, 20);
  run("dW LSTM 512x1024x2240", 512, 1024, 2240, true, true, true, 20);
  run("Gx 2752x1024x256", 2752, 1024, 256, false, true, true, 20);
  return 0;
}
