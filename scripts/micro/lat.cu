// microbenchmarks: dependent-chain latencies on sm_100a (diagnostics only)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0, t1;
  __syncthreads();
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 0.5);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // div chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = y / (x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // shfl chain (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // barrier chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // smem load chain (pointer chase)
  __shared__ int sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x & 1023;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = sm[p];
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
  // FFMA chain (fp32)
  float fx = (float)a, fy = (float)b;
  t0 = clock64();
  for (int i = 0; i < n; ++i) fx = fmaf(fx, fy, 0.5f);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = t1 - t0;
  out[threadIdx.x] = x + p + fx;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64 * 8);
  const char* names[] = {"dfma", "dadd", "ddiv", "dsqrt", "shfl.f64", "bar.sync", "lds.chase", "ffma"};
  int threads[] = {32, 512, 1024};
  for (int ti = 0; ti < 3; ++ti) {
    for (int rep = 0; rep < 2; ++rep) {
      k<<<1, threads[ti]>>>(out, cyc, 0.999, 0.5, 1000);
      cudaDeviceSynchronize();
    }
    printf("threads=%d:", threads[ti]);
    for (int i = 0; i < 8; ++i) printf(" %s=%.1f", names[i], cyc[i] / 1000.0);
    printf("\n");
  }
  return 0;
}
