// Host cost per call of the C ABI's small forward vs a bare kernel launch
// (dev tool): nvcc -o tools/launch_probe tools/launch_probe.cu -Lpaper_2509_10613_b200/_native -lsigkernel
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "../include/sigkernel.h"

__global__ void empty_kernel(double* p) {
  if (threadIdx.x == 1000) p[0] = 1.0;
}

int main() {
  const int B = 32, L = 64, d = 4;
  std::vector<double> h(B * L * d);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 0.001 * (double)(i % 97);
  double *x, *y, *out;
  cudaMalloc(&x, h.size() * 8);
  cudaMalloc(&y, h.size() * 8);
  cudaMalloc(&out, B * 8);
  cudaMemcpy(x, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(y, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  auto bench = [&](const char* name, auto fn) {
    for (int i = 0; i < 100; ++i) fn();
    cudaStreamSynchronize(st);
    const int n = 20;
    auto t0 = std::chrono::high_resolution_clock::now();
    for (int i = 0; i < n; ++i) fn();
    auto t1 = std::chrono::high_resolution_clock::now();
    cudaStreamSynchronize(st);
    auto t2 = std::chrono::high_resolution_clock::now();
    printf("%-28s host %.2f us/call, drain %.2f us\n", name,
           std::chrono::duration<double, std::micro>(t1 - t0).count() / n,
           std::chrono::duration<double, std::micro>(t2 - t1).count());
  };
  bench("empty kernel launch", [&] { empty_kernel<<<32, 128, 0, st>>>(out); });
  bench("empty kernel 80KB smem", [&] {
    static bool once = [] {
      cudaFuncSetAttribute((const void*)empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      return true;
    }();
    (void)once;
    empty_kernel<<<32, 128, 80 * 1024, st>>>(out);
  });
  bench("sk_forward_batch (C1)", [&] {
    sk_forward_batch(x, y, B, L, L, d, 0, 0, SK_STATIC_LINEAR, 1.0, out, nullptr, 0, st);
  });
  cudaError_t e = cudaGetLastError();
  printf("last error: %s, sk_last_error: %s\n", cudaGetErrorString(e), sk_last_error());
  return 0;
}
