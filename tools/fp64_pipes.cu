// Microbenchmark: fp64 FMA-pipe vs DMMA (mma.sync m8n8k4 f64) throughput on one
// B200, alone and interleaved (do they share a pipe?).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_pipes tools/fp64_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters) {
  double f[8];
  for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
  double c[4][2] = {};
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
    }
    if (MODE & 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += f[i];
  for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, grid = 148 * 4, block = 256;
  const char* names[] = {"", "dfma only", "dmma only", "both"};
  for (int mode = 1; mode <= 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 1) k<1><<<grid, block>>>(d, iters);
      if (mode == 2) k<2><<<grid, block>>>(d, iters);
      if (mode == 3) k<3><<<grid, block>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double thr = (double)grid * block * iters;
      const double fma_dfma = (mode & 1) ? thr * 32 : 0;       // 32 DFMA per thread-iter
      const double fma_dmma = (mode & 2) ? thr / 32 * 4 * 256 : 0;   // 4 DMMA per warp-iter, 256 FMA each
      if (rep) printf("%-10s %8.3f ms  dfma %.2f TFMA/s  dmma %.2f TFMA/s  total %.2f TFLOP/s\n", names[mode], ms,
                      fma_dfma / ms / 1e9, fma_dmma / ms / 1e9, 2 * (fma_dfma + fma_dmma) / ms / 1e9);
    }
  }
  return 0;
}
