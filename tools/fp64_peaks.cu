// fp64_peaks.cu -- measures the FP64 roofline denominators on the box:
//   DFMA issue rate (the path's bound), DMMA (mma.sync f64),
//   DFMA+DMMA interleaved (are they separate pipes?), SHFL rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void dfma_kernel(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, double a, double b) {
  double c[8][2];
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = threadIdx.x + j;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mixed_kernel(double* out, double a, double b) {
  double c[4][2];
  for (int j = 0; j < 4; ++j) c[j][0] = c[j][1] = threadIdx.x + j;
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma(c[j][0], c[j][1], a, b);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void shfl_kernel(double* out, int seed) {
  int v0 = threadIdx.x ^ seed, v1 = v0 + 1, v2 = v0 + 2, v3 = v0 + 3;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v0 = __shfl_up_sync(0xffffffffu, v0, 1); v1 = __shfl_up_sync(0xffffffffu, v1, 1);
      v2 = __shfl_up_sync(0xffffffffu, v2, 1); v3 = __shfl_up_sync(0xffffffffu, v3, 1);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v0 + v1 + v2 + v3;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  float ms;
  auto time_it = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5.0;
  };
  double t = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3); });
  double dfma = (double)blocks * threads * ITERS * 32 / (t * 1e-3);
  printf("{\"sms\": %d, \"clock_khz\": %d,\n", sms, clk);
  printf(" \"dfma_per_s\": %.4e, \"dfma_tflops\": %.2f,\n", dfma, 2 * dfma / 1e12);
  t = time_it([&] { dmma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3); });
  double dmma_fma = (double)blocks * (threads / 32) * ITERS * 8 * 256 / (t * 1e-3);
  printf(" \"dmma_fma_per_s\": %.4e, \"dmma_tflops\": %.2f,\n", dmma_fma, 2 * dmma_fma / 1e12);
  t = time_it([&] { mixed_kernel<<<blocks, threads>>>(out, 0.999, 1e-3); });
  double mixed = ((double)blocks * (threads / 32) * ITERS * 4 * 256 +
                  (double)blocks * threads * ITERS * 16) / (t * 1e-3);
  printf(" \"mixed_fma_per_s\": %.4e, \"mixed_ms\": %.3f,\n", mixed, t);
  t = time_it([&] { shfl_kernel<<<blocks, threads>>>(out, 3); });
  double shfl = (double)blocks * threads * ITERS * 16 / (t * 1e-3);
  printf(" \"shfl_lanes_per_s\": %.4e}\n", shfl);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
