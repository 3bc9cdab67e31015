// Host cost of a kernel launch: <<<>>> vs cudaLaunchKernelEx with / without
// the programmatic-stream-serialization attribute.  Diagnostic only.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

struct Args {
  const float* const* p;
  int n, m;
  float x[8];
};

__global__ void empty_kernel(Args a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.n == -12345) printf("x");
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  Args a{};
  a.n = 1;
  auto bench = [&](const char* name, auto fn) {
    for (int i = 0; i < 200; ++i) fn();
    cudaStreamSynchronize(s);
    const int N = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) fn();
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t2 = std::chrono::steady_clock::now();
    printf("%-28s host %.2f us/launch, device-drain %.2f us/launch\n", name,
           std::chrono::duration<double, std::micro>(t1 - t0).count() / N,
           std::chrono::duration<double, std::micro>(t2 - t0).count() / N);
  };
  bench("<<<>>>", [&] { empty_kernel<<<148, 256, 0, s>>>(a); });
  for (int pdl = 0; pdl < 2; ++pdl) {
    bench(pdl ? "LaunchKernelEx + PDL" : "LaunchKernelEx", [&] {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = pdl;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, empty_kernel, a);
    });
  }
  return 0;
}
