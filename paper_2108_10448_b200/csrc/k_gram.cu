// k_gram.cu -- fp64 Gram matrix of each mode's intersection on its short side.
//
// The reference factorises every intersection C_i(I_i, :) (|I_i| x |J_i|) with
// a full Householder + implicit-QR SVD (linalg.py:59-74 -> _core.pyx:24-58).
// On the device we only need its rank-r_i truncation, so each intersection B
// (viewed as s x l, s = min(|I|, |J|)) is reduced to the s x s Gram K = B B^T
// (this kernel), whose top-r eigenvectors give the short-side singular
// subspace (k_eig.cu); the long-side vectors, the singular values and the
// orthonormality repair are then recomputed directly from B (k_svdpost.cu), so
// singular values keep absolute accuracy ~eps*sigma_1 as in the reference.
#include "common.cuh"

#define GRAM_T 64      // output tile edge
#define GRAM_KS 16     // k-step


struct GramArgs {
  const int* stop;   // the engine's stop flag (iteration launches), or null
  int n;
  int s[RT_MAX_MODES];
  i64 l[RT_MAX_MODES];
  int tall[RT_MAX_MODES];           // 1: B = M^T (|I| > |J|), else B = M
  i64 mrows[RT_MAX_MODES];          // rows of M (= |I_k|)
  const double* M[RT_MAX_MODES];
  double* part;                     // [n][maxchunks][maxpairs][T*T]
  double* K[RT_MAX_MODES];          // packed lower s(s+1)/2
  double* Kfull[RT_MAX_MODES];      // optional mirrored s x s copy (row-major), or null
  int maxchunks, maxpairs;
  int cl;                           // long-side chunk per CTA (split-K), multiple of GRAM_KS
};

__device__ __forceinline__ double gram_B(const GramArgs& ga, int k, i64 a, i64 t) {
  const double* M = ga.M[k];
  return ga.tall[k] ? M[t + a * ga.mrows[k]] : M[a + t * ga.mrows[k]];
}

__device__ __forceinline__ void pair_decode(int pair, int& I, int& J) {
  int i = (int)((sqrt(8.0 * pair + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= pair) ++i;
  while (i * (i + 1) / 2 > pair) --i;
  I = i;
  J = pair - i * (i + 1) / 2;
}

__global__ void __launch_bounds__(256) k_gram_tiles(GramArgs ga) {
  if (rt_stopped(ga.stop)) return;
  const int k = blockIdx.z;
  if (k >= ga.n) return;
  const int s = ga.s[k];
  const i64 l = ga.l[k];
  const int nt = (s + GRAM_T - 1) / GRAM_T;
  const int npairs = nt * (nt + 1) / 2;
  const int pair = blockIdx.x;
  if (pair >= npairs) return;
  const i64 t0 = (i64)blockIdx.y * ga.cl;
  if (t0 >= l) return;
  const i64 t1 = min(l, t0 + ga.cl);
  int I, J;
  pair_decode(pair, I, J);
  __shared__ double As[2][GRAM_KS][GRAM_T + 1];
  __shared__ double Bs[2][GRAM_KS][GRAM_T + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  // register-prefetched double buffer: the next k-step's loads are in flight
  // while the current one is multiplied
  constexpr int PER = GRAM_T * GRAM_KS / 256;   // elements per thread per operand
  double pa[PER], pb[PER];
  auto fetch = [&](i64 tt) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + u * 256;
      const int r = idx % GRAM_T, kk = idx / GRAM_T;
      const i64 t = tt + kk;
      const int a = I * GRAM_T + r, b = J * GRAM_T + r;
      pa[u] = (a < s && t < t1) ? gram_B(ga, k, a, t) : 0.0;
      pb[u] = (b < s && t < t1) ? gram_B(ga, k, b, t) : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + u * 256;
      const int r = idx % GRAM_T, kk = idx / GRAM_T;
      As[buf][kk][r] = pa[u];
      Bs[buf][kk][r] = pb[u];
    }
  };
  fetch(t0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (i64 tt = t0; tt < t1; tt += GRAM_KS) {
    const bool more = tt + GRAM_KS < t1;
    if (more) fetch(tt + GRAM_KS);
#pragma unroll
    for (int kk = 0; kk < GRAM_KS; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[buf][kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  double* out = ga.part + (((i64)k * ga.maxchunks + blockIdx.y) * ga.maxpairs + pair) * (GRAM_T * GRAM_T);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) out[(ty * 4 + i) * GRAM_T + tx + 16 * j] = acc[i][j];
}

// The same 64 x 64 split-K tiles on the fp64 tensor cores: mma.sync m8n8k4 f64
// (DMMA).  4 warps as 2 x 2, each a 32 x 32 sub-tile = 4 x 4 mma tiles (32 fp64
// accumulators per thread); per k-step of 4: 4 A and 4 B fragments (one double per
// lane each) feed 16 DMMAs.  Fragment layout (PTX m8n8k4 .f64, row.col):
//   A[g][t], B[t][g], C[g][2t + {0,1}], g = lane / 4, t = lane % 4.
// Shared rows padded to 68 doubles (the 4 k-rows of a fragment load hit distinct
// banks).  Partials go to the same layout as k_gram_tiles (k_gram_reduce sums them).
#define GRAM_LDS 68
__global__ void __launch_bounds__(128) k_gram_tiles_dmma(GramArgs ga) {
  if (rt_stopped(ga.stop)) return;
  const int k = blockIdx.z;
  if (k >= ga.n) return;
  const int s = ga.s[k];
  const i64 l = ga.l[k];
  const int nt = (s + GRAM_T - 1) / GRAM_T;
  const int npairs = nt * (nt + 1) / 2;
  const int pair = blockIdx.x;
  if (pair >= npairs) return;
  const i64 t0 = (i64)blockIdx.y * ga.cl;
  if (t0 >= l) return;
  const i64 t1 = min(l, t0 + ga.cl);
  int I, J;
  pair_decode(pair, I, J);
  __shared__ __align__(16) double As[2][GRAM_KS][GRAM_LDS];
  __shared__ __align__(16) double Bs[2][GRAM_KS][GRAM_LDS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = (w >> 1) * 32, wc = (w & 1) * 32;   // warp sub-tile origin
  const int g = lane >> 2, tq = lane & 3;
  double c[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  constexpr int PER = GRAM_T * GRAM_KS / 128;   // elements per thread per operand
  double pa[PER], pb[PER];
  auto fetch = [&](i64 tt) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + u * 128;
      const int r = idx % GRAM_T, kk = idx / GRAM_T;
      const i64 t = tt + kk;
      const int a = I * GRAM_T + r, b = J * GRAM_T + r;
      pa[u] = (a < s && t < t1) ? gram_B(ga, k, a, t) : 0.0;
      pb[u] = (b < s && t < t1) ? gram_B(ga, k, b, t) : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + u * 128;
      const int r = idx % GRAM_T, kk = idx / GRAM_T;
      As[buf][kk][r] = pa[u];
      Bs[buf][kk][r] = pb[u];
    }
  };
  fetch(t0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (i64 tt = t0; tt < t1; tt += GRAM_KS) {
    const bool more = tt + GRAM_KS < t1;
    if (more) fetch(tt + GRAM_KS);
#pragma unroll
    for (int ks = 0; ks < GRAM_KS; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][ks + tq][wr + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][ks + tq][wc + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(c[i][j][0]), "+d"(c[i][j][1])
                       : "d"(af[i]), "d"(bf[j]));
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  double* out = ga.part + (((i64)k * ga.maxchunks + blockIdx.y) * ga.maxpairs + pair) * (GRAM_T * GRAM_T);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2* o = reinterpret_cast<double2*>(out + (wr + i * 8 + g) * GRAM_T + wc + j * 8 + 2 * tq);
      *o = make_double2(c[i][j][0], c[i][j][1]);
    }
}

// Sum the split-K partials (warp per output, fixed butterfly order) into packed lower K.
__global__ void __launch_bounds__(256) k_gram_reduce(GramArgs ga) {
  if (rt_stopped(ga.stop)) return;
  const int k = blockIdx.y;
  if (k >= ga.n) return;
  const int s = ga.s[k];
  const i64 npk = (i64)s * (s + 1) / 2;
  const int nchunks = (int)((ga.l[k] + ga.cl - 1) / ga.cl);
  const int lane = threadIdx.x & 31;
  for (i64 idx = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < npk;
       idx += ((i64)gridDim.x * blockDim.x) >> 5) {
    int i = (int)((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
    while ((i64)(i + 1) * (i + 2) / 2 <= idx) ++i;
    while ((i64)i * (i + 1) / 2 > idx) --i;
    const int j = (int)(idx - (i64)i * (i + 1) / 2);
    const int I = i / GRAM_T, J = j / GRAM_T;
    const int pair = I * (I + 1) / 2 + J;
    const int li = i % GRAM_T, lj = j % GRAM_T;
    const double* p = ga.part + ((i64)k * ga.maxchunks * ga.maxpairs + pair) * (GRAM_T * GRAM_T) + li * GRAM_T + lj;
    double acc = 0.0;
    for (int c = lane; c < nchunks; c += 32) acc += p[(i64)c * ga.maxpairs * (GRAM_T * GRAM_T)];
    acc = warp_sum(acc);
    if (lane == 0) {
      ga.K[k][idx] = acc;
      if (ga.Kfull[k]) {   // the mirrored s x s copy (row-contiguous matvecs of the Lanczos path)
        ga.Kfull[k][(i64)i * s + j] = acc;
        ga.Kfull[k][(i64)j * s + i] = acc;
      }
    }
  }
}
