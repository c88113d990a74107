// dmma_probe.cu -- what exactly does mma.sync.m8n8k4.f64 compute, and how fast?
//   1. arithmetic: compare D = A*B + C from DMMA with candidate fma orders
//   2. throughput: DMMA alone, DFMA alone, and interleaved
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// A row-major 8x4, B col-major (B[k][n] at n*4+k), C/D 8x8 row-major
__global__ void one_mma(const double* A, const double* B, const double* C, double* D) {
  int l = threadIdx.x;
  int g = l >> 2, t = l & 3;
  double a = A[g * 4 + t];
  double b = B[g * 4 + t];  // B[k=t][n=g]
  double c0 = C[g * 8 + 2 * t], c1 = C[g * 8 + 2 * t + 1];
  double d0, d1;
  dmma(d0, d1, a, b, c0, c1);
  D[g * 8 + 2 * t] = d0;
  D[g * 8 + 2 * t + 1] = d1;
}

template <int MODE>
__global__ void thr(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2];
  double f[16];
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int i = 0; i < 16; ++i) f[i] = i * 0.5;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b, c[i][0], c[i][1]);
    }
    if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int r = 0; r < (MODE == 2 ? 4 : 8); ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], b, a);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < 16; ++i) s += f[i];
  if (s == 12345.678) out[0] = s;
}

static double rnd() { return (double)rand() / RAND_MAX * 2.0 - 1.0; }

int main() {
  double hA[32], hB[32], hC[64], hD[64];
  double *A, *B, *C, *D;
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512); cudaMalloc(&D, 512);
  int ok_seq = 0, ok_rev = 0, ok_exact = 0, ok_pairs = 0, total = 0;
  for (int trial = 0; trial < 2000; ++trial) {
    for (int i = 0; i < 32; ++i) { hA[i] = rnd() * pow(2.0, rand() % 40 - 20); hB[i] = rnd() * pow(2.0, rand() % 40 - 20); }
    for (int i = 0; i < 64; ++i) hC[i] = (trial % 2) ? 0.0 : rnd();
    cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(C, hC, 512, cudaMemcpyHostToDevice);
    one_mma<<<1, 32>>>(A, B, C, D);
    cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
    for (int m = 0; m < 8; ++m)
      for (int n = 0; n < 8; ++n) {
        double a[4], b[4];
        for (int k = 0; k < 4; ++k) { a[k] = hA[m * 4 + k]; b[k] = hB[n * 4 + k]; }
        double c = hC[m * 8 + n];
        double s = c;
        for (int k = 0; k < 4; ++k) s = fma(a[k], b[k], s);
        double r = c;
        for (int k = 3; k >= 0; --k) r = fma(a[k], b[k], r);
        long double e = c;
        for (int k = 0; k < 4; ++k) e += (long double)a[k] * b[k];
        double p = fma(a[1], b[1], a[0] * b[0]) + fma(a[3], b[3], a[2] * b[2]) + c;
        double got = hD[m * 8 + n];
        ok_seq += got == s; ok_rev += got == r; ok_exact += got == (double)e; ok_pairs += got == p;
        ++total;
      }
  }
  printf("DMMA arithmetic over %d outputs: seq-fma k0..3 %d, reverse-fma %d, exact(long double) %d, pairwise %d\n",
         total, ok_seq, ok_rev, ok_exact, ok_pairs);

  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps = 4; warps <= 16; warps *= 2) {
      dim3 grid(sms * 2), block(32 * warps);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) thr<0><<<grid, block>>>(out, iters);
        if (mode == 1) thr<1><<<grid, block>>>(out, iters);
        if (mode == 2) thr<2><<<grid, block>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double nw = (double)grid.x * warps;
        double fma_dmma = (mode == 0 || mode == 2) ? nw * iters * 8 * 256 : 0;
        double fma_dfma = (mode == 1) ? nw * iters * 8 * 16 * 32 : (mode == 2 ? nw * iters * 4 * 16 * 32 : 0);
        if (rep == 1)
          printf("mode %s warps/CTA %2d: %.3f ms, DMMA %.3e FMA/s, DFMA %.3e FMA/s, total %.3e FMA/s\n",
                 mode == 0 ? "dmma" : mode == 1 ? "dfma" : "mix ", warps, ms, fma_dmma / ms * 1e3,
                 fma_dfma / ms * 1e3, (fma_dmma + fma_dfma) / ms * 1e3);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
