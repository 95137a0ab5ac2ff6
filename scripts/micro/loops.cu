// diagnostics: cycles of the eigensolver inner loops in isolation
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2108_10448_b200/csrc/common.cuh"
extern "C" unsigned long long rtcur_launch_counter_add(unsigned long long k) { return k; }
#include "../../paper_2108_10448_b200/csrc/k_eig.cu"

__global__ void kst(long long* cyc, int s, int* out) {
  __shared__ double d[256], e2[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) { d[i] = i < s ? 0.5 + 0.001 * i : 1e30; e2[i] = i + 1 < s ? 0.01 : 0.0; }
  __syncthreads();
  long long t0 = clock64();
  int c = 0;
  int s4 = 1 + ((s - 1 + 3) / 4) * 4;
  for (int rep = 0; rep < 10; ++rep) { int c0, c1; sturm_count2(d, e2, s4, 0.3 + 0.01 * threadIdx.x + rep * 1e-3, 0.31 + 0.01 * threadIdx.x, c0, c1); c += c0 + c1; }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 10;
  out[threadIdx.x] = c;
}

__global__ void kupd(long long* cyc, int L, double* sink) {
  extern __shared__ double sm[];
  const int ld = L | 1;
  double* A = sm;
  double* vc = A + L * ld;
  double* yy = vc + L;
  for (int i = threadIdx.x; i < L * ld; i += blockDim.x) A[i] = 1.0 / (1 + i);
  for (int i = threadIdx.x; i < L; i += blockDim.x) { vc[i] = 0.1 * i; yy[i] = 0.2; }
  __syncthreads();
  const int sub = threadIdx.x & 3, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double kk = 0.01, v0 = 0.3;
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    for (int ib = wid * 8; ib < L; ib += nw * 8) {
      const int i = ib + lane / 4;
      if (i < L) {
        const double vi = i == 0 ? v0 : vc[i];
        const double wi = yy[i] - kk * vi;
        double* row = A + i * ld;
        for (int j = sub; j < L; j += 4) {
          const double vj = j == 0 ? v0 : vc[j];
          row[j] = row[j] - (vi * (yy[j] - kk * vj) + wi * vj);
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 10;
  sink[threadIdx.x] = A[threadIdx.x];
}

int main() {
  long long* cyc; int* out; double* sink;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&out, 4096); cudaMalloc(&sink, 8192 * 8);
  for (int s : {42, 90, 213}) {
    kst<<<1, 32>>>(cyc, s, out); cudaDeviceSynchronize();
    kst<<<1, 32>>>(cyc, s, out); cudaDeviceSynchronize();
    printf("sturm s=%d: %lld cycles/count (%.1f per step)\n", s, cyc[0], (double)cyc[0] / s);
  }
  cudaFuncSetAttribute(kupd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int L : {41, 89, 150}) {
    size_t smb = ((size_t)L * (L | 1) + 2 * L) * 8;
    kupd<<<1, 512, smb>>>(cyc, L, sink); cudaDeviceSynchronize();
    kupd<<<1, 512, smb>>>(cyc, L, sink); cudaDeviceSynchronize();
    printf("update L=%d: %lld cycles (%s)\n", L, cyc[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
