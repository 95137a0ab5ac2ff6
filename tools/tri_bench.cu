// tri_bench.cu -- micro-benchmark of Householder tridiagonalisation designs for the
// eigensolver's full path (k_eig.cu), s <= 128, full storage in shared memory:
//   variant 0: one warp does everything (no block barriers, lanes own rows)
//   variant 1: four warps (one per SM sub-partition), named barriers
// Outputs d (s), e (s-1) and the clock64 span; correctness is checked from
// Python (tools/tri_bench.py) against numpy's eigenvalues.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/_tri_bench.so tools/tri_bench.cu
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one warp; A full storage (ld odd), rows owned cyclically by lanes (<= 4 rows each)
template <int NR>
__device__ void tri_warp(double* A, int ld, int s, double* d, double* e, double* vs, double* ws) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k + 2 < s; ++k) {
    const int b0 = k + 1, L = s - b0;
    const double* rowk = A + k * ld;
    double sq = 0.0;
    for (int j = b0 + lane; j < s; j += 32) sq = fma(rowk[j], rowk[j], sq);
    const double nrm = sqrt(wsum(sq));
    const double x0 = rowk[b0];
    double alpha = 0.0, beta = 0.0;
    if (nrm > 0.0) {
      alpha = -copysign(nrm, x0);
      beta = 1.0 / (nrm * (nrm + fabs(x0)));
    }
    for (int j = b0 + lane; j < s; j += 32) vs[j] = (j == b0) ? x0 - alpha : rowk[j];
    __syncwarp();
    // y_i = beta * sum_j A[i][j] v_j for the lane's rows
    double y[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) y[q] = 0.0;
    for (int j = b0; j < s; ++j) {
      const double vj = vs[j];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int i = b0 + lane + 32 * q;
        if (i < s) y[q] = fma(A[i * ld + j], vj, y[q]);
      }
    }
    double dp = 0.0;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int i = b0 + lane + 32 * q;
      y[q] *= beta;
      if (i < s) dp = fma(y[q], vs[i], dp);
    }
    const double kk = 0.5 * beta * wsum(dp);
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int i = b0 + lane + 32 * q;
      if (i < s) ws[i] = y[q] - kk * vs[i];
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int i = b0 + lane + 32 * q;
      if (i < s) {
        const double vi = vs[i], wi = ws[i];
        double* row = A + i * ld;
        for (int j = b0; j < s; ++j) row[j] -= vi * ws[j] + wi * vs[j];
      }
    }
    if (lane == 0) {
      d[k] = A[k * ld + k];
      e[k] = alpha;
    }
    __syncwarp();
    (void)L;
  }
  if (lane == 0) {
    d[s - 2] = A[(s - 2) * ld + s - 2];
    e[s - 2] = A[(s - 1) * ld + s - 2];
    d[s - 1] = A[(s - 1) * ld + s - 1];
  }
}

// four warps (128 threads), rows cyclic over threads, named barrier 1
template <int NR>
__device__ void tri_4w(double* A, int ld, int s, double* d, double* e, double* vs, double* ws, double* part) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  for (int k = 0; k + 2 < s; ++k) {
    const int b0 = k + 1;
    const double* rowk = A + k * ld;
    // every warp computes the reflector redundantly (no barrier for the norm)
    double sq = 0.0;
    for (int j = b0 + lane; j < s; j += 32) sq = fma(rowk[j], rowk[j], sq);
    const double nrm = sqrt(wsum(sq));
    const double x0 = rowk[b0];
    double alpha = 0.0, beta = 0.0;
    if (nrm > 0.0) {
      alpha = -copysign(nrm, x0);
      beta = 1.0 / (nrm * (nrm + fabs(x0)));
    }
    double* vw = vs + wid * 128;   // per-warp copy of v
    for (int j = b0 + lane; j < s; j += 32) vw[j] = (j == b0) ? x0 - alpha : rowk[j];
    __syncwarp();
    double y[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) y[q] = 0.0;
    for (int j = b0; j < s; ++j) {
      const double vj = vw[j];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int i = b0 + t + 128 * q;
        if (i < s) y[q] = fma(A[i * ld + j], vj, y[q]);
      }
    }
    double dp = 0.0;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int i = b0 + t + 128 * q;
      y[q] *= beta;
      if (i < s) dp = fma(y[q], vw[i], dp);
    }
    dp = wsum(dp);
    double* pk = part + (k & 1) * 4;
    if (lane == 0) pk[wid] = dp;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int i = b0 + t + 128 * q;
      if (i < s) ws[i] = y[q];   // y now; w formed after the barrier
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const double kk = 0.5 * beta * (((pk[0] + pk[1]) + pk[2]) + pk[3]);
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int i = b0 + t + 128 * q;
      if (i < s) {
        const double vi = vw[i], wi = y[q] - kk * vi;
        double* row = A + i * ld;
        for (int j = b0; j < s; ++j) row[j] -= vi * (ws[j] - kk * vw[j]) + wi * vw[j];
      }
    }
    if (t == 0) {
      d[k] = A[k * ld + k];
      e[k] = alpha;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
  }
  if (t == 0) {
    d[s - 2] = A[(s - 2) * ld + s - 2];
    e[s - 2] = A[(s - 1) * ld + s - 2];
    d[s - 1] = A[(s - 1) * ld + s - 1];
  }
}

extern __shared__ double smem[];

__global__ void k_tri(const double* K, int s, int variant, double* d, double* e, long long* cyc) {
  const int ld = s | 1;
  double* A = smem;
  double* vs = A + s * ld;       // 4 x 128
  double* ws = vs + 512;         // 128
  double* part = ws + 128;       // 8
  for (int x = threadIdx.x; x < s * s; x += blockDim.x) A[(x / s) * ld + (x % s)] = K[x];
  __syncthreads();
  long long t0 = clock64();
  if (variant == 0) {
    if (threadIdx.x < 32) {
      if (s <= 64) tri_warp<2>(A, ld, s, d, e, vs, ws);
      else tri_warp<4>(A, ld, s, d, e, vs, ws);
    }
  } else {
    if (threadIdx.x < 128) tri_4w<1>(A, ld, s, d, e, vs, ws, part);
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = clock64() - t0;
}

extern "C" int tri_run(const double* K, int s, int variant, double* d, double* e, long long* cyc) {
  const int ld = s | 1;
  const size_t sm = (size_t)(s * ld + 512 + 128 + 8) * 8;
  cudaFuncSetAttribute(k_tri, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  k_tri<<<1, 512, sm>>>(K, s, variant, d, e, cyc);
  return (int)cudaDeviceSynchronize();
}
