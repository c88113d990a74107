// Dependent-chain latencies on this GPU (dev tool): DFMA, DADD, SHFL (double),
// LDS (double), one warp, clock64 around 1024-long chains.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = lane * 0.5; sm[lane + 32] = 0.0;
  __syncwarp();
  double x = a;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) x = fma(x, b, a);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) x = x + b;
  long long t2 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) x = __shfl_up_sync(0xffffffffu, x, 1) + 0.0;
  long long t3 = clock64();
  int idx = lane;
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) idx = (int)sm[idx & 63] + lane;
  long long t4 = clock64();
  out[lane] = x + idx;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}

int main() {
  double* out; long long* cyc; cudaMalloc(&out, 256); cudaMallocManaged(&cyc, 64);
  for (int r = 0; r < 3; ++r) { probe<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999); cudaDeviceSynchronize(); }
  printf("cycles per dependent op: DFMA %.1f  DADD %.1f  SHFL+DADD %.1f  LDS.64+cvt+IADD %.1f\n",
         cyc[0] / 1024.0, cyc[1] / 1024.0, cyc[2] / 1024.0, cyc[3] / 1024.0);
  return 0;
}
