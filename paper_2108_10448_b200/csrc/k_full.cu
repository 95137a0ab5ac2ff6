// k_full.cu -- K3: streaming full-tensor reconstruction + threshold + residual
// sums, the device form of the reference's full-output step
//   L = cur_reconstruct_full(cur)              (cli.py:238 -> fiber_cur.py:277-285)
//   S = hard_threshold(x - L, zeta_final)       (cli.py:240-242)
// evaluated in Tucker form L(i_1, R) = sum_a A_1[i_1, a] Tf[R, a] with
// Tf = G x_{m>=2} A_m (one fp64 row of r_1 values per mode-1 fiber), so each
// element costs r_1 FMAs and the kernel streams X once and writes L and S once
// (3 E bytes per element).  Works on a mode-1 slab [lo, hi) of a sharded X.
#include "full_types.cuh"


template <typename T>
__global__ void __launch_bounds__(256) k_full(FullArgs a) {
  __shared__ double red[8];
  __shared__ bool am_last;
  const i64 ld = a.hi - a.lo;
  const i64 n = ld * a.ncols;
  const T* X = reinterpret_cast<const T*>(a.X);
  T* L = reinterpret_cast<T*>(a.L);
  T* S = reinterpret_cast<T*>(a.S);
  double e2 = 0.0, x2 = 0.0;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const double* A1 = a.A1 + a.lo;
  // each thread walks elements e = start + k*stride; (i1, col) tracked incrementally
  i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (e < n) {
    i64 col = e / ld, i1 = e - col * ld;
    const i64 dcol = stride / ld, di = stride - dcol * ld;
    for (; e < n; e += stride) {
      const double x = X ? (double)X[e] : 0.0;
      const double* tf = a.Tf + col * a.r1;
      double l = 0.0;
      for (int k = 0; k < a.r1; ++k) l = fma(A1[i1 + k * a.d1], tf[k], l);
      const double s = hard_thr(x - l, a.zeta);
      const double res = x - l - s;
      e2 = fma(res, res, e2);
      x2 = fma(x, x, x2);
      if (L) L[e] = (T)l;
      if (S) S[e] = (T)s;
      i1 += di;
      col += dcol;
      if (i1 >= ld) { i1 -= ld; ++col; }
    }
  }
  e2 = block_sum(e2, red);
  x2 = block_sum(x2, red);
  if (threadIdx.x == 0) {
    a.partial[2 * blockIdx.x] = e2;
    a.partial[2 * blockIdx.x + 1] = x2;
    __threadfence();
    am_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double se = 0.0, sx = 0.0;
  for (i64 t = threadIdx.x; t < gridDim.x; t += blockDim.x) {
    se += ((volatile double*)a.partial)[2 * t];
    sx += ((volatile double*)a.partial)[2 * t + 1];
  }
  se = block_sum(se, red);
  sx = block_sum(sx, red);
  if (threadIdx.x == 0) {
    a.sums[0] = se;
    a.sums[1] = sx;
    *a.counter = 0u;
  }
}

template __global__ void k_full<float>(FullArgs);
template __global__ void k_full<double>(FullArgs);

// ------------------------------------------------------------------ synthetic instances

// Counter-based uniform in [0, 1) keyed by (seed, global element index, stream).
__device__ __forceinline__ double gen_u01(unsigned long long seed, unsigned long long idx, unsigned long long stream) {
  unsigned long long z = seed * 0x9E3779B97F4A7C15ull + idx * 0xD1B54A32D192ED03ull + stream * 0x8CB92BA72F3D8DD7ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

// X = L + S on a mode-1 slab [lo, hi): S is Bernoulli(alpha) supported with
// values U[-cmu, cmu], both drawn from the GLOBAL element index, so any slab
// decomposition of the tensor reproduces the same instance (BASELINE configs,
// SURVEY §8(d.1)).  L (fp64) may alias nothing; X is written in dtype.
template <typename T>
__global__ void __launch_bounds__(256) k_gen_outliers(const double* __restrict__ L, T* __restrict__ X, i64 nloc, i64 lo,
                                                      i64 hi, i64 d1, unsigned long long seed, double alpha,
                                                      double cmu) {
  const i64 ld = hi - lo;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < nloc; e += (i64)gridDim.x * blockDim.x) {
    const i64 R = e / ld, i1 = e - R * ld;
    const unsigned long long gidx = (unsigned long long)(lo + i1 + d1 * R);
    double v = L[e];
    if (gen_u01(seed, gidx, 1) < alpha) v += (2.0 * gen_u01(seed, gidx, 2) - 1.0) * cmu;
    X[e] = (T)v;
  }
}
template __global__ void k_gen_outliers<float>(const double*, float*, i64, i64, i64, i64, unsigned long long, double,
                                               double);
template __global__ void k_gen_outliers<double>(const double*, double*, i64, i64, i64, i64, unsigned long long,
                                                double, double);

// Generator pass over a mode-1 slab [lo, hi): L(i1, R) = sum_a Y1[i1, a] Tf[R, a]
// (Y1: d1 x r1 column-major, Tf: ncols x r1 row-major, both shared by every slab,
// so each entry is bitwise independent of the slab decomposition).
//   mode 0: sums |L| over the slab (per-CTA partials, last CTA sums in order)
//   mode 1: writes X = L + S (hashed outliers, values U[-cmu, cmu]) in T
template <typename T>
__global__ void __launch_bounds__(256) k_gen_tucker(const double* __restrict__ Y1, const double* __restrict__ Tf,
                                                    i64 d1, int r1, i64 lo, i64 hi, i64 ncols, int mode,
                                                    unsigned long long seed, double alpha, double cmu,
                                                    T* __restrict__ X, double* partial, double* out_sum,
                                                    unsigned int* counter) {
  __shared__ double red[8];
  __shared__ bool am_last;
  const i64 ld = hi - lo;
  const i64 n = ld * ncols;
  double acc = 0.0;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
    const i64 R = e / ld, i1 = e - R * ld;
    const double* tf = Tf + R * r1;
    double l = 0.0;
    for (int a = 0; a < r1; ++a) l = fma(Y1[lo + i1 + (i64)a * d1], tf[a], l);
    if (mode == 0) {
      acc += fabs(l);
    } else {
      const unsigned long long gidx = (unsigned long long)(lo + i1 + d1 * R);
      if (gen_u01(seed, gidx, 1) < alpha) l += (2.0 * gen_u01(seed, gidx, 2) - 1.0) * cmu;
      X[e] = (T)l;
    }
  }
  if (mode != 0) return;
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = acc;
    __threadfence();
    am_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double t = 0.0;
  for (i64 c = threadIdx.x; c < gridDim.x; c += blockDim.x) t += ((volatile double*)partial)[c];
  t = block_sum(t, red);
  if (threadIdx.x == 0) {
    *out_sum = t;
    *counter = 0u;
  }
}
template __global__ void k_gen_tucker<float>(const double*, const double*, i64, int, i64, i64, i64, int,
                                             unsigned long long, double, double, float*, double*, double*,
                                             unsigned int*);
template __global__ void k_gen_tucker<double>(const double*, const double*, i64, int, i64, i64, i64, int,
                                              unsigned long long, double, double, double*, double*, double*,
                                              unsigned int*);
