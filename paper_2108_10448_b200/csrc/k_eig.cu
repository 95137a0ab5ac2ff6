// k_eig.cu -- top-r eigenvectors of a small symmetric PSD matrix (the
// intersection Gram, s <= 235), one CTA per matrix, fp64 throughout, all
// working data in shared memory:
//
//   1. Householder tridiagonalisation K = Q T Q^T.  Small s: full symmetric
//      storage (odd leading dimension, conflict-free rows), row groups of 8
//      threads for the symv and the rank-2 update, reflectors copied to a
//      contiguous array.  Large s (full storage does not fit 227 KB): packed
//      lower triangle, warp per row, reflectors kept in place.  3 barriers per
//      Householder step in both layouts.
//   2. The r largest eigenvalues of T by multisection on Sturm counts of the
//      tn-normalised T (one warp per eigenvalue, 32 shifts per round; the
//      three-term recurrence runs branch-free in groups of 4 with exact
//      power-of-two rescaling in between).
//   3. Block inverse iteration on T: thread-per-vector pivoted tridiagonal LU
//      (factored once, 3 solves); vectors whose eigenvalues cluster (gap below
//      1e-3 * ||T||, LAPACK dstein's ORTOL) are re-orthogonalised after every
//      solve, everything once more (CGS2) at the end.
//   4. Back-transform by the stored reflectors, warp per vector (no barriers).
//
// Only the span of the r vectors must be accurate: the Rayleigh-Ritz step in
// k_svdpost.cu fixes the basis inside it and recomputes the singular values
// from the intersection itself.  Replaces the dense_svd call of linalg.py:73
// (_core.pyx:24-249) for the rank-r part the solver uses.
#include "common.cuh"
#include <cfloat>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define EIG_SMEM_DOUBLES 29056   // 227 KB opt-in shared memory per CTA
#define EIG_TPR 4                // threads per row group (full-storage path)
#define EIG_THREADS 512
#define EIG_CLUSTER 8            // CTAs per mode for 128 < s <= 256 (register-tiled tridiagonalisation)

struct EigArgs {
  const int* stop;   // the engine's stop flag (iteration launches), or null
  int n;
  int s[RT_MAX_MODES];
  int r[RT_MAX_MODES];
  const double* K[RT_MAX_MODES];   // packed lower, s(s+1)/2
  double* E[RT_MAX_MODES];         // s x r, column-major (output)
  double* lam[RT_MAX_MODES];       // r, descending (output)
  int nb[RT_MAX_MODES];            // inverse-iteration batch (vectors factored at once)
  int full[RT_MAX_MODES];          // 1: full-storage tridiagonalisation
  long long* tmark;                // optional: per-matrix clock64 marks at phase boundaries (8 each)
  // warm start for the subspace-iteration fast path (null: full solver only)
  int lz_stride;                       // Lanczos: Ritz extraction every lz_stride steps from max(16, 3r)
  const double* Kfull[RT_MAX_MODES];   // packed storage: the mirrored s x s Gram in global memory (Lanczos matvec), or null
  const double* warmA[RT_MAX_MODES];   // previous iterate's A_k (d_k x r_k, column-major)
  const int* warm_rows[RT_MAX_MODES];  // current row set I_k (0-based)
  i64 warm_d[RT_MAX_MODES];
  int max_sub_steps;
  int ms_warps;                        // multisection: max warps per eigenvalue (shifts = 64 x warps)
  int* fast_used;                      // per mode: 1 if the fast path certified the subspace
  int reg_tridiag;                     // register-tiled tridiagonalisation: 1 for 128 < s <= 256 (clusters), 2 also s <= 128
  // Lanczos full path (s <= 128, full storage): Krylov basis capacity (0: off) and
  // its shared-memory offset (doubles from the start of the dynamic smem)
  int lz_mcap[RT_MAX_MODES];
  int lz_off[RT_MAX_MODES];
  // inverse-iteration LU factors in global scratch (r x 4s doubles, then r x s
  // pivot bytes), or null: in shared memory, nb at a time.  Used when fewer than
  // r factorisations fit next to K (s = 213 packed: 2), so all r run at once.
  double* lug[RT_MAX_MODES];
};

__host__ __device__ inline int eig_ld(int s) { return s | 1; }

// doubles of shared memory k_eig needs for (s, r, nb, layout).  The full solver's
// tail arrays (T's diagonals, reflector scratch, inverse-iteration LU) are idle
// during the warm subspace iteration, so its scratch (Y: s x r, three r x r)
// aliases them and only the excess (sub) is extra.
__host__ __device__ inline long long eig_tail_doubles(int s, int nb) {
  return 8LL * s + 8 + (long long)nb * 4 * s + ((long long)nb * s + 7) / 8 + 8;
}
__host__ __device__ inline long long eig_smem_doubles(int s, int r, int nb, int full, int sub = 0) {
  const long long amat = full ? (long long)s * eig_ld(s) + (long long)s * (s - 1) / 2 : (long long)s * (s + 1) / 2;
  const long long need = (long long)s * r + 3LL * r * r, tail = eig_tail_doubles(s, nb);
  return amat + (long long)s * r + 2LL * r + 96 + tail + (sub && need > tail ? need - tail : 0);
}

// Lanczos basis capacity for the full path (0: not used): full storage, 64 <= s <=
// 128 (below 64 the Householder path's s - 2 steps are no more than the ~24 Lanczos
// steps plus Ritz checks: measured 1.63 vs 1.70 ms per solve at s = 42), basis
// columns up to 64 and within the 227 KB next to the base layout
#define EIG_LZ_MMAX 64
__host__ __device__ inline int eig_lz_mcap(int s, int r, long long base_doubles, int full) {
  if (s < 64 || s > 256 || (full && s > 128)) return 0;
  // full storage: after the base layout; packed: over the shared-memory copy of K
  const long long avail = full ? EIG_SMEM_DOUBLES - base_doubles - 8 : (long long)s * (s + 1) / 2;
  long long m = full ? avail / (s + 2) - 1 : avail / s - 1;   // full: basis + 2 coefficient vectors
  m = m < EIG_LZ_MMAX ? m : EIG_LZ_MMAX;
  m = m < s - 1 ? m : s - 1;
  return m >= (3 * r > 12 ? 3 * r : 12) ? (int)m : 0;
}

__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }  // i >= j

__device__ __forceinline__ double hash_unit(unsigned long long a) {
  a += 0x9E3779B97F4A7C15ull;
  a = (a ^ (a >> 30)) * 0xBF58476D1CE4E5B9ull;
  a = (a ^ (a >> 27)) * 0x94D049BB133111EBull;
  a ^= a >> 31;
  return (double)(a >> 11) * (2.0 / 9007199254740992.0) - 1.0;   // (-1, 1)
}

// Number of eigenvalues of the normalised tridiagonal (d, e2 = offdiag^2, all
// entries O(1); arrays padded to a multiple of 4 with d = +1e30, e2 = 0, which
// adds no sign change) strictly less than x0 and x1 (two independent Sturm
// sequences interleaved for ILP): sign changes of the leading principal minors,
// a zero minor replaced by -tiny * previous (the q-form's -pivmin), rescaled by
// an exact power of two every 4 steps.
__device__ __forceinline__ void sturm_count2(const double* __restrict__ d, const double* __restrict__ e2, int s4,
                                             double x0, double x1, int& c0, int& c1) {
  const double tiny = 1e-300;
  double pa1 = d[0] - x0, pb1 = d[0] - x1, pa2 = 1.0, pb2 = 1.0;
  pa1 = (pa1 == 0.0) ? -tiny : pa1;
  pb1 = (pb1 == 0.0) ? -tiny : pb1;
  int ca = pa1 < 0.0, cb = pb1 < 0.0;
  bool na = pa1 < 0.0, nb = pb1 < 0.0;
  for (int i = 1; i < s4; i += 4) {
    double dv[4], ev[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { dv[u] = d[i + u]; ev[u] = e2[i + u - 1]; }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double pa = fma(dv[u] - x0, pa1, -ev[u] * pa2);
      double pb = fma(dv[u] - x1, pb1, -ev[u] * pb2);
      pa = (pa == 0.0) ? -tiny * pa1 : pa;
      pb = (pb == 0.0) ? -tiny * pb1 : pb;
      const bool qa = pa < 0.0, qb = pb < 0.0;
      ca += (qa != na);
      cb += (qb != nb);
      na = qa;
      nb = qb;
      pa2 = pa1; pa1 = pa;
      pb2 = pb1; pb1 = pb;
    }
    const int ea = (int)((__double_as_longlong(pa1) >> 52) & 0x7ff);
    const int eb = (int)((__double_as_longlong(pb1) >> 52) & 0x7ff);
    if (ea > 1023 + 300 || ea < 1023 - 300) {
      const double sc = __longlong_as_double((long long)(2046 - ea) << 52);   // 2^(1023-ea), exact
      pa1 *= sc;
      pa2 *= sc;
    }
    if (eb > 1023 + 300 || eb < 1023 - 300) {
      const double sc = __longlong_as_double((long long)(2046 - eb) << 52);
      pb1 *= sc;
      pb2 *= sc;
    }
  }
  c0 = ca;
  c1 = cb;
}

// sum over the warp of red[0..nw) (every lane gets the total; deterministic order)
__device__ __forceinline__ double warp_sum_of(const double* red, int nw) {
  const int lane = threadIdx.x & 31;
  double t = lane < nw ? red[lane] : 0.0;
  return warp_sum(t);
}

__device__ __forceinline__ double group_sum8(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

// ---------------------------------------------------------------- subspace iteration
// Top-r invariant subspace of the PSD Gram K (resident in shared memory, full or
// packed) by block power iteration from a warm start X0 = A_prev(I, :), with
// Cholesky-QR (twice) orthonormalisation.  Certified when
//     ||K X - X H||_F <= 1e-12 * delta,   delta = lambda_min(H) - (tr K - tr H)
// where H = X^T K X: for PSD K every eigenvalue outside the top r is at most
// tr K - tr(top-r) <= tr K - tr H, so delta lower-bounds the spectral gap and
// the subspace angle is <= 1e-12 (Davis-Kahan sin-theta).  Returns false
// (caller falls back to the full solver) otherwise.  Block-uniform result.
__device__ __forceinline__ double eig_kval(const double* A, bool full, int ld, int i, int j) {
  return full ? A[i * ld + j] : (i >= j ? A[pk(i, j)] : A[pk(j, i)]);
}

// In-place lower Cholesky of the r x r symmetric C (column-major, r <= 32) by
// warp 0, lane i owning row i: C = L L^T with L in the lower triangle and the
// reciprocal diagonal in rinv[0..r).  Every pivot must exceed `floor` (else
// false).  Call with the whole block; returns a block-uniform result.
__device__ bool eig_chol_warp(double* C, int r, double* rinv, double floor, double* scal) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 32) {
    bool ok = true;
    for (int k = 0; k < r; ++k) {
      // pivot (row k, already updated by the previous columns)
      const double piv = C[k + k * r];
      if (!(piv > floor)) { ok = false; break; }
      const double d = sqrt(piv), di = 1.0 / d;
      if (lane == k) { C[k + k * r] = d; rinv[k] = di; }
      double lik = 0.0;
      if (lane > k && lane < r) {
        lik = C[lane + k * r] * di;
        C[lane + k * r] = lik;
      }
      __syncwarp();
      // trailing update of row `lane`: C[lane, j] -= L[lane, k] L[j, k], k < j <= lane
      if (lane > k && lane < r)
        for (int j = k + 1; j <= lane; ++j) C[lane + j * r] = fma(-lik, C[j + k * r], C[lane + j * r]);
      __syncwarp();
    }
    if (lane == 0) scal[8] = ok ? 1.0 : 0.0;
  }
  __syncthreads();
  return scal[8] != 0.0;
}

// Cholesky-QR of X (s x r, column-major): X <- X L^-T.  false if not SPD.
__device__ bool eig_cholqr(double* X, int s, int r, double* C, double* rinv, double* scal) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int np = r * (r + 1) / 2;
  for (int q = wid; q < np; q += nw) {
    int a = 0, rem = q;
    while (rem >= r - a) { rem -= r - a; ++a; }
    const int b = a + rem;
    double d = 0.0;
    for (int i = lane; i < s; i += 32) d = fma(X[a * s + i], X[b * s + i], d);
    d = warp_sum(d);
    if (lane == 0) { C[a + b * r] = d; C[b + a * r] = d; }
  }
  __syncthreads();
  if (!eig_chol_warp(C, r, rinv, 1e-28 * C[0], scal)) return false;
  // rows: y L^T = x  (forward substitution, reciprocal pivots), in place column by
  // column: entries k < j of the thread's row are already the solved ones
  for (int i = tid; i < s; i += blockDim.x) {
    for (int j = 0; j < r; ++j) {
      double v = X[j * s + i];
      for (int k = 0; k < j; ++k) v = fma(-X[k * s + i], C[j + k * r], v);
      X[j * s + i] = v * rinv[j];
    }
  }
  __syncthreads();
  return true;
}

__device__ bool eig_subspace(const double* A, bool full, int ld, int s, int r, double* X, double* Y, double* H,
                             double* C, double* Rm, double* red, double* red2, double* scal, const double* warmA,
                             const int* rows, i64 d, int max_steps, long long* tmk) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
#define TMK(j) if (tmk && tid == 0 && step == 1) tmk[j] = clock64();
  double* rinv = Rm;   // r reciprocal pivots
  // trace and squared Frobenius norm of K, and the warm start
  double t = 0.0, f2 = 0.0;
  for (int i = tid; i < s; i += blockDim.x) t += eig_kval(A, full, ld, i, i);
  if (full) {
    for (int e = tid; e < s * s; e += blockDim.x) {
      const double v = A[(e / s) * ld + (e % s)];
      f2 = fma(v, v, f2);
    }
  } else {
    // packed rows by warps, lanes across the row (off-diagonal entries count twice)
    for (int i = wid; i < s; i += nw) {
      const double* row = A + pk(i, 0);
      for (int j = lane; j <= i; j += 32) {
        const double v = row[j];
        f2 = fma(v, v * (j == i ? 1.0 : 2.0), f2);
      }
    }
  }
  t = warp_sum(t);
  f2 = warp_sum(f2);
  if (lane == 0) {
    red[wid] = t;
    red2[wid] = f2;
  }
  for (int e = tid; e < s * r; e += blockDim.x) {
    const int i = e % s, c = e / s;
    X[e] = warmA[rows[i] + (i64)c * d];
  }
  __syncthreads();
  const double trK = warp_sum_of(red, nw);
  const double kf2 = warp_sum_of(red2, nw);
  if (!(trK > 0.0)) return false;
  __syncthreads();
  for (int rep = 0; rep < 2; ++rep)
    if (!eig_cholqr(X, s, r, C, rinv, scal)) return false;
  const int nch = (r + 3) >> 2;   // 4-column chunks
  for (int step = 0; step < max_steps; ++step) {
    TMK(2)
    // Y = K X: item (row i, 4-column chunk), each K element read once per chunk
    for (int it = tid; it < s * nch; it += blockDim.x) {
      const int ch = it / s, i = it - ch * s;
      const int c0 = ch * 4;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const double* x0 = X + c0 * s;
      const bool h1 = c0 + 1 < r, h2 = c0 + 2 < r, h3 = c0 + 3 < r;
      if (full) {
        const double* row = A + i * ld;
        for (int j = 0; j < s; ++j) {
          const double k = row[j];
          a0 = fma(k, x0[j], a0);
          if (h1) a1 = fma(k, x0[s + j], a1);
          if (h2) a2 = fma(k, x0[2 * s + j], a2);
          if (h3) a3 = fma(k, x0[3 * s + j], a3);
        }
      } else {
        // row part j <= i (contiguous packed row), column part j > i (column i of rows j)
        const double* row = A + pk(i, 0);
        for (int j = 0; j <= i; ++j) {
          const double k = row[j];
          a0 = fma(k, x0[j], a0);
          if (h1) a1 = fma(k, x0[s + j], a1);
          if (h2) a2 = fma(k, x0[2 * s + j], a2);
          if (h3) a3 = fma(k, x0[3 * s + j], a3);
        }
        int cb = pk(i + 1, i);
        for (int j = i + 1; j < s; ++j) {
          const double k = A[cb];
          cb += j + 1;
          a0 = fma(k, x0[j], a0);
          if (h1) a1 = fma(k, x0[s + j], a1);
          if (h2) a2 = fma(k, x0[2 * s + j], a2);
          if (h3) a3 = fma(k, x0[3 * s + j], a3);
        }
      }
      double* y0 = Y + c0 * s + i;
      y0[0] = a0;
      if (h1) y0[s] = a1;
      if (h2) y0[2 * s] = a2;
      if (h3) y0[3 * s] = a3;
    }
    __syncthreads();
    TMK(3)
    // H = X^T Y (symmetrised)
    const int np = r * (r + 1) / 2;
    for (int q = wid; q < np; q += nw) {
      int a = 0, rem = q;
      while (rem >= r - a) { rem -= r - a; ++a; }
      const int b = a + rem;
      double d1 = 0.0, d2 = 0.0;
      for (int i = lane; i < s; i += 32) {
        d1 = fma(X[a * s + i], Y[b * s + i], d1);
        d2 = fma(X[b * s + i], Y[a * s + i], d2);
      }
      const double hv = 0.5 * (warp_sum(d1) + warp_sum(d2));
      if (lane == 0) { H[a + b * r] = hv; H[b + a * r] = hv; }
    }
    __syncthreads();
    // residual ||Y - X H||_F^2 and ||Y||_F^2
    double rn = 0.0, yn = 0.0;
    for (int e = tid; e < s * r; e += blockDim.x) {
      const int i = e % s, c = e / s;
      const double y = Y[e];
      double v = y;
      for (int k = 0; k < r; ++k) v -= X[k * s + i] * H[k + c * r];
      rn = fma(v, v, rn);
      yn = fma(y, y, yn);
    }
    rn = warp_sum(rn);
    yn = warp_sum(yn);
    if (lane == 0) {
      red2[wid] = rn;
      red[wid] = yn;
    }
    __syncthreads();
    const double res = sqrt(warp_sum_of(red2, nw));
    const double yf2 = warp_sum_of(red, nw);
    // forecast: from the two-step decay rate of the residual, give up (full solver)
    // when more further steps would be needed to reach the certification level than
    // the full path costs
    if (step >= 3) {
      const double prev2 = scal[12 + (step & 1)];
      const double rho2 = res / prev2;   // per two steps
      bool hopeless = !(rho2 < 0.5);
      if (!hopeless) {
        const double target = 1e-13 * trK;   // certification needs res ~ 1e-12 * gap
        // the full path's cost grows with s: allow ~s/8 more steps (4..10)
        const double budget = fmin(10.0, fmax(4.0, s / 8.0));
        if (res > target) hopeless = 0.5 * log(target / res) / log(rho2) > budget;
      }
      if (hopeless) return false;
    }
    __syncthreads();
    TMK(4)
    if (tid == 0) scal[12 + (step & 1)] = res;
    if (tid == 0) scal[14] = (double)(step + 1);
    double trH = 0.0, hf2 = 0.0;
    for (int c = 0; c < r; ++c) trH += H[c + c * r];
    for (int e = 0; e < r * r; ++e) hf2 = fma(H[e], H[e], hf2);
    // Rigorous upper bound u >= lambda_{r+1}(K): Courant-Fischer with V = span X gives
    // lambda_{r+1} <= lambda_max((I-P)K(I-P)) <= ||(I-P)K(I-P)||_F, and
    // ||(I-P)K(I-P)||_F^2 = ||K||_F^2 - 2||KX||_F^2 + ||X^T K X||_F^2 (X orthonormal),
    // plus a rounding margin for the three fixed-order sums; for PSD K also
    // lambda_{r+1} <= tr K - tr H.  Take the smaller.
    const double fro = sqrt(fmax(kf2 - 2.0 * yf2 + hf2, 0.0) + 4.0 * (double)s * s * DBL_EPSILON * kf2);
    const double ub = fmin(trK - trH, fro);
    // lambda_min(H) <= tr H / r: if even that cannot exceed the bound, certification
    // is impossible from this subspace -> give up at once (full solver)
    if (!(trH / r - ub > 0.0)) return false;
    // certify: lambda_min(H) > mu = ub + 1e12 res  <=>  H - mu I is positive definite
    // (one warp Cholesky of the shifted copy; no eigen-solve needed); then the
    // subspace angle is <= res / (lambda_min(H) - ub) <= 1e-12 (Davis-Kahan)
    if (res <= 1e-9 * trK) {
      const double mu = ub + 1e12 * res;
      double* Hs = C;   // scratch (C is re-formed by the next Cholesky-QR)
      for (int e = tid; e < r * r; e += blockDim.x) Hs[e] = H[e] - ((e % r == e / r) ? mu : 0.0);
      __syncthreads();
      if (eig_chol_warp(Hs, r, rinv, 0.0, scal)) return true;
    }
    // Long attempt, nearly converged, bound settled (within 1e-3 of the previous
    // step's): once lambda_min(H) <= min_i H_ii lies below 0.95 ub no later step
    // can certify (the Frobenius bound is too loose for this spectrum) -> full
    // solver now rather than at max_steps.
    const double ub_prev = scal[15];
    __syncthreads();   // (every thread has read scal[15])
    if (tid == 0) scal[15] = ub;
    if (step >= 5 && res <= 1e-8 * trK && fabs(ub - ub_prev) <= 1e-3 * ub) {
      double hmin = H[0];
      for (int c = 1; c < r; ++c) hmin = fmin(hmin, H[c + c * r]);
      if (hmin < 0.95 * ub) return false;
    }
    if (step + 1 == max_steps) break;
    TMK(5)
    // X <- orth(Y)
    for (int e = tid; e < s * r; e += blockDim.x) X[e] = Y[e];
    __syncthreads();
    for (int rep = 0; rep < 2; ++rep)
      if (!eig_cholqr(X, s, r, C, rinv, scal)) return false;
    TMK(6)
  }
  return false;
}

// ---------------------------------------------------------------- register-tiled tridiagonalisation
// Householder tridiagonalisation with K held in REGISTERS: warp w owns rows
// i = w + 16a (a < RB), lane l owns columns j = l + 32b (b < CB) (cyclic, so the
// shrinking trailing block stays balanced).  Per step the only shared-memory
// traffic is O(s) vectors: the reflected column (written by its owners during
// the previous step's update, with its squared-norm partials), the symv result
// y (one writer lane per row after a transpose-reduce over the warp's lanes)
// and the dot partials -- 2 barriers per step, RB*CB + 2*RB*CB FMAs per thread.
// The shared-memory version below it reads and rewrites the whole trailing
// block from shared memory every step (bandwidth/latency bound).  Outputs are
// identical in layout: reflectors contiguous in HV (step k: s-k-1 entries,
// v_0 = x_0 - alpha), dd / ed / bet, and the trailing 2x2 block in dd/ed.
// Returns hoff (total reflector length).
template <int RB>
__device__ __forceinline__ double eig_xpose_reduce(double (&v)[RB], int lane) {
  // reduce RB per-lane values over the 32 lanes: after the call the lane holds the
  // full sum of row index eig_xpose_row<RB>(lane) (fixed shuffle tree)
  if constexpr (RB >= 8) {
    const bool up = lane & 16;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double send = up ? v[t] : v[t + 4], keep = up ? v[t + 4] : v[t];
      v[t] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  if constexpr (RB >= 4) {
    constexpr int o = RB >= 8 ? 8 : 16;
    const bool up = lane & o;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double send = up ? v[t] : v[t + 2], keep = up ? v[t + 2] : v[t];
      v[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  if constexpr (RB >= 2) {
    constexpr int o = RB >= 8 ? 4 : RB >= 4 ? 8 : 16;
    const bool up = lane & o;
    const double send = up ? v[0] : v[1], keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, o);
  }
  double t = v[0];
  constexpr int first = RB >= 8 ? 2 : RB >= 4 ? 4 : RB >= 2 ? 8 : 16;
#pragma unroll
  for (int o = first; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

template <int RB>
__device__ __forceinline__ int eig_xpose_row(int lane) {
  if constexpr (RB >= 8) return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  else if constexpr (RB >= 4) return ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
  else if constexpr (RB >= 2) return (lane >> 4) & 1;
  else return 0;
}

// C == 1: one CTA, K read from its shared-memory full storage (A, ld).  C > 1: a
// cluster of C CTAs, CTA c owning the rows of global warps 16c..16c+15, K read
// from the packed global Gram (Kg); the per-step vectors and partials are
// broadcast into every CTA's shared memory (DSMEM stores) and the two barriers
// are cluster barriers.  dd / ed / bet / HV are written to CTA 0 (which goes on
// with the eigenvalues); red holds 2 x 16C norm partials, red2 16C dot partials.
template <int C>
__device__ __forceinline__ void eig_csync() {
  if constexpr (C == 1) __syncthreads();
  else cg::this_cluster().sync();
}
// p[0] = v in CTA `rank`'s copy of this shared-memory location (C == 1: local store).
// mapa + st.shared::cluster per store: 32-bit addresses recomputed on the spot keep
// register pressure down (hoisted generic remote pointers spill next to the tile)
template <int C>
__device__ __forceinline__ void eig_put(double* p, int rank, double v) {
  if constexpr (C == 1) {
    *p = v;
  } else {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    unsigned ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
  }
}

template <int C, int RB, int CB>
__device__ int eig_tridiag_reg(const double* __restrict__ A, int ld, const double* __restrict__ Kg, int s,
                               double* HV, double* dd, double* ed, double* bet, double* xs0, double* xs1, double* ys,
                               double* red, double* red2) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int crank = 0;
  if constexpr (C > 1) crank = (int)cg::this_cluster().block_rank();
  constexpr int NP = 16 * C;            // row-owning warps in the cluster
  const int gw = crank * 16 + wid;
  double kr[RB][CB];
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int i = gw + NP * a, j = lane + 32 * b;
      double v = 0.0;
      if (i < s && j < s) {
        if constexpr (C == 1) v = A[i * ld + j];
        else v = i >= j ? Kg[pk(i, j)] : Kg[pk(j, i)];
      }
      kr[a][b] = v;
    }
  // column 0 below the diagonal: its owners (lane 0, b = 0) publish it with its norm partials
  if (lane == 0) {
    double sq = 0.0;
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      const int i = gw + NP * a;
      if (i >= 1 && i < s) {
#pragma unroll
        for (int c2 = 0; c2 < C; ++c2) eig_put<C>(xs0 + i, c2, kr[a][0]);
        sq = fma(kr[a][0], kr[a][0], sq);
      }
    }
#pragma unroll
    for (int c2 = 0; c2 < C; ++c2) eig_put<C>(red + gw, c2, sq);
  }
  eig_csync<C>();
  constexpr int WL = 32 / RB;           // lanes sharing one reduced row (writer: lane % WL == 0)
  const int arow = eig_xpose_row<RB>(lane);
  int hoff = 0;
  for (int k = 0; k + 2 < s; ++k) {
    const double* xc = (k & 1) ? xs1 : xs0;
    double* xn = (k & 1) ? xs0 : xs1;
    const double* rc = red + (k & 1) * NP;
    double* rn = red + ((k + 1) & 1) * NP;
    double t0 = 0.0;
    for (int q = lane; q < NP; q += 32) t0 += rc[q];
    const double nrm = sqrt(warp_sum(t0));
    const double x0 = xc[k + 1];
    double alpha = 0.0, beta = 0.0;
    if (nrm > 0.0) {
      alpha = -copysign(nrm, x0);
      beta = 1.0 / (nrm * (nrm + fabs(x0)));
    }
    const double v0 = x0 - alpha;
    double vcol[CB];
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int j = lane + 32 * b;
      vcol[b] = (j > k && j < s) ? (j == k + 1 ? v0 : xc[j]) : 0.0;
    }
    // y = beta K22 v for this warp's rows
    double pr[RB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      double t = 0.0;
#pragma unroll
      for (int b = 0; b < CB; ++b) t = fma(kr[a][b], vcol[b], t);
      pr[a] = t;
    }
    const double ysum = beta * eig_xpose_reduce<RB>(pr, lane);
    double dotp = 0.0;
    {
      const int i = gw + NP * arow;
      if ((lane % WL) == 0 && i > k && i < s) {
#pragma unroll
        for (int c2 = 0; c2 < C; ++c2) eig_put<C>(ys + i, c2, ysum);
        dotp = ysum * (i == k + 1 ? v0 : xc[i]);
      }
    }
    dotp = warp_sum(dotp);
    if (lane == 0) {
#pragma unroll
      for (int c2 = 0; c2 < C; ++c2) eig_put<C>(red2 + gw, c2, dotp);
    }
    // the reflector (CTA 0, warp 0: every CTA holds all columns) and the step's scalars
    if (crank == 0 && wid == 0) {
#pragma unroll
      for (int b = 0; b < CB; ++b) {
        const int j = lane + 32 * b;
        if (j > k && j < s) HV[hoff + j - k - 1] = vcol[b];
      }
    }
    if (crank == 0 && tid == 0) {
      ed[k] = alpha;
      bet[k] = beta;
    }
    if (gw == (k % NP) && lane == (k & 31)) {
      // select chains (no dynamic register indexing: that would move kr to local memory)
      const int ak = k / NP, bk = k >> 5;
      double pick = 0.0;
#pragma unroll
      for (int a = 0; a < RB; ++a)
#pragma unroll
        for (int b = 0; b < CB; ++b) pick = (a == ak && b == bk) ? kr[a][b] : pick;
      eig_put<C>(dd + k, 0, pick);
    }
    eig_csync<C>();                                                // B1
    double t1 = 0.0;
    for (int q = lane; q < NP; q += 32) t1 += red2[q];
    const double kk = 0.5 * beta * warp_sum(t1);
    double wcol[CB];
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int j = lane + 32 * b;
      wcol[b] = (j > k && j < s) ? ys[j] - kk * vcol[b] : 0.0;
    }
    // K22 -= v w^T + w v^T; the next step's column (k+1, rows > k+1) goes out with its norm
    const int kn = k + 1;
    double sq = 0.0;
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      const int i = gw + NP * a;
      const bool act = i > k && i < s;
      const double vi = act ? (i == k + 1 ? v0 : xc[i]) : 0.0;
      const double wi = act ? ys[i] - kk * vi : 0.0;
#pragma unroll
      for (int b = 0; b < CB; ++b) kr[a][b] -= vi * wcol[b] + wi * vcol[b];
      if (lane == (kn & 31) && i > kn && i < s) {
        const int bn = kn >> 5;
        double x = 0.0;
#pragma unroll
        for (int b = 0; b < CB; ++b) x = (b == bn) ? kr[a][b] : x;
#pragma unroll
        for (int c2 = 0; c2 < C; ++c2) eig_put<C>(xn + i, c2, x);
        sq = fma(x, x, sq);
      }
    }
    if (lane == (kn & 31)) {
#pragma unroll
      for (int c2 = 0; c2 < C; ++c2) eig_put<C>(rn + gw, c2, sq);
    }
    hoff += s - k - 1;
    eig_csync<C>();                                                // B2
  }
  // trailing 2x2 block: K[s-2][s-2], K[s-1][s-2], K[s-1][s-1] -> CTA 0
  {
    double p22 = 0.0, p12 = 0.0, p11 = 0.0;
    bool h22 = false, h12 = false, h11 = false;
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) {
        const int i = gw + NP * a, j = lane + 32 * b;
        const bool c22 = i == s - 2 && j == s - 2, c12 = i == s - 1 && j == s - 2, c11 = i == s - 1 && j == s - 1;
        p22 = c22 ? kr[a][b] : p22;
        p12 = c12 ? kr[a][b] : p12;
        p11 = c11 ? kr[a][b] : p11;
        h22 |= c22;
        h12 |= c12;
        h11 |= c11;
      }
    if (h22) eig_put<C>(dd + s - 2, 0, p22);
    if (h12) eig_put<C>(ed + s - 2, 0, p12);
    if (h11) eig_put<C>(dd + s - 1, 0, p11);
  }
  eig_csync<C>();
  return hoff;
}

extern __shared__ double eig_smem[];

// The r largest eigenpairs of the symmetric tridiagonal T (dd: diagonal, ed:
// off-diagonal, size s) into E (s x r, column-major, stride s): multisection on
// Sturm counts of the tn-normalised T, then block inverse iteration with cluster
// re-orthogonalisation and a final CGS2 (see the header).  Used on the
// Householder tridiagonal (s = |I_k|) and on the Lanczos tridiagonal T_m.
// scal[1], scal[2]: Gershgorin bounds of T; tn > 0 its norm bound.
__device__ void eig_tri_vectors(const EigArgs& ea, int mi, int s, int r, int nb, double tn, const double* dd,
                                const double* ed, double* dn, double* e2n, double* lam, int* clus, double* red,
                                double* red2, const double* scal, double* lu, unsigned char* piv, double* E,
                                long long* tm) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  // ---------------------------------------------------------------- 2. multisection (normalised T)
  const double itn = 1.0 / tn;
  const int s4 = 1 + ((s - 1 + 3) / 4) * 4;   // padded length of the Sturm arrays
  for (int i = tid; i < s4; i += blockDim.x) {
    dn[i] = i < s ? dd[i] * itn : 1e30;
    const double en = (i + 1 < s) ? ed[i] * itn : 0.0;
    e2n[i] = en * en;
  }
  __syncthreads();
  {
    // ng warps per eigenvalue test ng*32 shifts per round; brackets combined in
    // shared memory (double-buffered by round parity: one barrier per round)
    const double pad = 4.0 * DBL_EPSILON * s;
    double* blo = red;                  // 2 x 16 warp brackets (lo); red/red2 are free here
    double* bhi = red2;                 // 2 x 16 warp brackets (hi)
    for (int j0 = 0; j0 < r; j0 += nw) {
      const int rr = min(nw, r - j0);
      // the counts are fp64-pipe bound on this one SM: more shifts per round cost more
      // than the rounds they save beyond ~one warp per eigenvalue
      const int ng = max(1, min(nw / rr, ea.ms_warps));
      const int j = j0 + wid / ng, g = wid % ng;
      const bool act = wid < rr * ng;
      const double nsh = (double)(ng * 64 + 1);
      const int rounds = (int)ceil(log(16.0 / DBL_EPSILON) / log(nsh)) + 1;
      double lo = scal[1] * itn - pad, hi = scal[2] * itn + pad;
      for (int round = 0; round < rounds; ++round) {
        double nlo = -DBL_MAX, nhi = DBL_MAX;
        if (act && hi > lo) {
          const int target = s - 1 - j;   // ascending index of the j-th largest
          const double xa = lo + (hi - lo) * (double)(g * 64 + 2 * lane + 1) / nsh;
          const double xb = lo + (hi - lo) * (double)(g * 64 + 2 * lane + 2) / nsh;
          int ca, cb;
          sturm_count2(dn, e2n, s4, xa, xb, ca, cb);
          if (ca <= target) nlo = xa;
          if (cb <= target) nlo = xb;
          if (cb >= target + 1) nhi = xb;
          if (ca >= target + 1) nhi = xa;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          nlo = fmax(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
          nhi = fmin(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
        }
        double* bl = blo + (round & 1) * 16;
        double* bh = bhi + (round & 1) * 16;
        if (lane == 0) { bl[wid] = nlo; bh[wid] = nhi; }
        __syncthreads();
        if (act) {
          for (int q = 0; q < ng; ++q) {
            const int w2 = (wid / ng) * ng + q;
            if (bl[w2] != -DBL_MAX) lo = fmax(lo, bl[w2]);
            if (bh[w2] != DBL_MAX) hi = fmin(hi, bh[w2]);
          }
          if (lo > hi) lo = hi = 0.5 * (lo + hi);
        }
      }
      if (act && g == 0 && lane == 0) lam[j] = 0.5 * (lo + hi) * tn;
      __syncthreads();
    }
  }
  __syncthreads();
  if (tid == 0) {
    // clusters (descending order): j joins j-1 when the gap is below ORTOL * ||T||
    clus[0] = 0;
    for (int j = 1; j < r; ++j) clus[j] = (lam[j - 1] - lam[j] < 1e-3 * tn) ? clus[j - 1] : j;
  }
  for (int j = tid; j < r; j += blockDim.x) ea.lam[mi][j] = lam[j];
  __syncthreads();
  if (tm && tid == 0) tm[3] = clock64();

  // ---------------------------------------------------------------- 3. block inverse iteration
  const double tiny = DBL_EPSILON * tn;
  const double pertol = 10.0 * DBL_EPSILON * tn;
  double* const lug = ea.lug[mi];
  const int nbe = lug ? r : nb;
  for (int j0 = 0; j0 < r; j0 += nbe) {
    const int jn = min(nbe, r - j0);
    double* u0 = lug ? lug + (size_t)4 * s * tid : lu + (size_t)4 * s * tid;
    double* u1 = u0 + s;
    double* u2 = u1 + s;
    double* lm = u2 + s;
    unsigned char* pv = lug ? reinterpret_cast<unsigned char*>(lug + (size_t)4 * s * r) + (size_t)s * tid
                            : piv + (size_t)s * tid;
    if (tid < jn) {
      const int j = j0 + tid;
      double mu = lam[j];
      // separate (nearly) equal shifts so every factorisation is distinct
      for (int i = 0; i < j; ++i)
        if (fabs(lam[i] - mu) < pertol * (j - i)) mu = lam[i] - pertol * (j - i);
      double ca = dd[0] - mu, cb = (s > 1) ? ed[0] : 0.0;
      for (int i = 0; i + 1 < s; ++i) {
        const double na = dd[i + 1] - mu;
        const double nbv = (i + 2 < s) ? ed[i + 1] : 0.0;
        const double c = ed[i];
        if (fabs(ca) >= fabs(c)) {
          if (fabs(ca) < tiny) ca = copysign(tiny, ca);
          const double inv = 1.0 / ca;
          const double l = c * inv;
          u0[i] = inv;
          u1[i] = cb;
          u2[i] = 0.0;
          pv[i] = 0;
          lm[i] = l;
          ca = na - l * cb;
          cb = nbv;
        } else {
          const double inv = 1.0 / c;
          const double l = ca * inv;
          u0[i] = inv;
          u1[i] = na;
          u2[i] = nbv;
          pv[i] = 1;
          lm[i] = l;
          ca = cb - l * na;
          cb = -l * nbv;
        }
      }
      if (fabs(ca) < tiny) ca = copysign(tiny, ca);
      u0[s - 1] = 1.0 / ca;
      u1[s - 1] = 0.0;
      u2[s - 1] = 0.0;
      if (s >= 2) u2[s - 2] = 0.0;
      double* x = E + j * s;
      for (int i = 0; i < s; ++i) x[i] = hash_unit(((unsigned long long)j << 32) ^ (unsigned long long)i);
    }
    __syncthreads();
    bool any_cluster = false;
    for (int j = j0; j < j0 + jn; ++j) any_cluster |= (clus[j] != j);
    for (int it = 0; it < 3; ++it) {
      if (tid < jn) {
        double* __restrict__ x = E + (j0 + tid) * s;
        double bi = x[0];
        double bn = s > 1 ? x[1] : 0.0;
        double l_i = lm[0];
        bool p_i = s > 1 ? pv[0] : 0;
        for (int i = 0; i + 1 < s; ++i) {
          // prefetch the next step's operands before the dependent update
          const double bnn = (i + 2 < s) ? x[i + 2] : 0.0;
          const double lnx = (i + 2 < s) ? lm[i + 1] : 0.0;
          const bool pnx = (i + 2 < s) ? pv[i + 1] : 0;
          double b_lo = bi, b_hi = bn;
          if (p_i) { b_lo = bn; b_hi = bi; }
          x[i] = b_lo;
          bi = fma(-l_i, b_lo, b_hi);
          bn = bnn;
          l_i = lnx;
          p_i = pnx;
        }
        x[s - 1] = bi;
        double xn1 = 0.0, xn2 = 0.0, mx = 0.0;
        double xi = x[s - 1], a1 = u1[s - 1], a2 = u2[s - 1], a0 = u0[s - 1];
        for (int i = s - 1; i >= 0; --i) {
          const double xp = i > 0 ? x[i - 1] : 0.0;
          const double b1 = i > 0 ? u1[i - 1] : 0.0, b2 = i > 0 ? u2[i - 1] : 0.0, b0 = i > 0 ? u0[i - 1] : 0.0;
          double v = (xi - a1 * xn1 - a2 * xn2) * a0;
          v = isfinite(v) ? v : 0.0;
          x[i] = v;
          mx = fmax(mx, fabs(v));
          xn2 = xn1;
          xn1 = v;
          xi = xp; a1 = b1; a2 = b2; a0 = b0;
        }
        const double inv = mx > 0.0 ? 1.0 / mx : 0.0;
        for (int i = 0; i < s; ++i) x[i] *= inv;
      }
      __syncthreads();
      if (!any_cluster) continue;
      // orthogonalise each clustered vector against the earlier members of its cluster
      for (int j = j0; j < j0 + jn; ++j) {
        const int c0 = clus[j];
        if (c0 == j) continue;
        double* xj = E + j * s;
        for (int pass = 0; pass < 2; ++pass) {
          for (int i = c0 + wid; i < j; i += nw) {
            const double* xi = E + i * s;
            double d = 0.0;
            for (int t = lane; t < s; t += 32) d = fma(xi[t], xj[t], d);
            d = warp_sum(d);
            if (lane == 0) red[i - c0] = d;
          }
          __syncthreads();
          for (int t = tid; t < s; t += blockDim.x) {
            double v = xj[t];
            for (int i = c0; i < j; ++i) v = fma(-red[i - c0], E[t + i * s], v);
            xj[t] = v;
          }
          __syncthreads();
        }
        double nn = 0.0;
        for (int t = tid; t < s; t += blockDim.x) nn = fma(xj[t], xj[t], nn);
        nn = warp_sum(nn);
        if (lane == 0) red2[wid] = nn;
        __syncthreads();
        nn = warp_sum_of(red2, nw);
        const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
        for (int t = tid; t < s; t += blockDim.x) xj[t] = nn > 0.0 ? xj[t] * inv : (t == j % s ? 1.0 : 0.0);
        __syncthreads();
      }
    }
  }
  // final CGS2 over all r vectors (warp w owns vector j; dots against the finished ones)
  for (int j = 0; j < r; ++j) {
    double* xj = E + j * s;
    for (int pass = 0; pass < 2; ++pass) {
      if (j > 0) {
        for (int i = wid; i < j; i += nw) {
          const double* xi = E + i * s;
          double d = 0.0;
          for (int t = lane; t < s; t += 32) d = fma(xi[t], xj[t], d);
          d = warp_sum(d);
          if (lane == 0) red[i] = d;
        }
        __syncthreads();
        for (int t = tid; t < s; t += blockDim.x) {
          double v = xj[t];
          for (int i = 0; i < j; ++i) v = fma(-red[i], E[t + i * s], v);
          xj[t] = v;
        }
      }
      double nn = 0.0;
      for (int t = tid; t < s; t += blockDim.x) nn = fma(xj[t], xj[t], nn);
      nn = warp_sum(nn);
      __syncthreads();
      if (lane == 0) red2[wid] = nn;
      __syncthreads();
      nn = warp_sum_of(red2, nw);
      const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
      for (int t = tid; t < s; t += blockDim.x) xj[t] = nn > 0.0 ? xj[t] * inv : (t == j % s ? 1.0 : 0.0);
      __syncthreads();
    }
  }
  if (tm && tid == 0) tm[4] = clock64();

}

// Gershgorin bounds of the tridiagonal (dd, ed) of size n into scal[0..2]:
// tn = max row sum, lo, hi (thread 0)
__device__ __forceinline__ void eig_tri_bounds(const double* dd, const double* ed, int n, double* scal) {
  double tn = 0.0, lo = DBL_MAX, hi = -DBL_MAX;
  for (int i = 0; i < n; ++i) {
    const double rad = (i > 0 ? fabs(ed[i - 1]) : 0.0) + (i + 1 < n ? fabs(ed[i]) : 0.0);
    tn = fmax(tn, fabs(dd[i]) + rad);
    lo = fmin(lo, dd[i] - rad);
    hi = fmax(hi, dd[i] + rad);
  }
  scal[0] = tn;
  scal[1] = lo;
  scal[2] = hi;
}

__global__ void __launch_bounds__(EIG_THREADS, 1) k_eig(EigArgs ea) {
  if (rt_stopped(ea.stop)) return;   // (every CTA of every cluster: no cluster barrier is pending)
  // launched either one CTA per mode, or (some s > 128) as clusters of EIG_CLUSTER
  // CTAs per mode: the cluster's extra CTAs only join the register-tiled
  // tridiagonalisation of modes with 128 < s <= 256 (eig_tridiag_reg<4, ...>)
  const int csize = (int)cg::this_cluster().num_blocks();
  const int crank = csize > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int mi = blockIdx.x / csize;
  if (mi >= ea.n) return;
  const int s = ea.s[mi], r = ea.r[mi], nb = ea.nb[mi];
  const bool use_cl = csize == EIG_CLUSTER && s > 128 && s <= 256 && ea.reg_tridiag;
  if (crank != 0 && !use_cl) return;   // (never reaches a cluster barrier)
  const bool full = ea.full[mi] != 0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int ld = eig_ld(s);
  const int npk = s * (s + 1) / 2;
  double* A = eig_smem;                                            // matrix
  double* HV = full ? A + s * ld : A;                              // reflectors (full: contiguous)
  double* E = full ? HV + s * (s - 1) / 2 : A + npk;               // s x r eigenvector block
  double* lam = E + s * r;                                         // r eigenvalues
  int* clus = reinterpret_cast<int*>(lam + r);                     // r cluster starts (as doubles)
  double* red = lam + 2 * r;                                       // 32
  double* red2 = red + 32;                                         // 32
  double* scal = red2 + 32;                                        // 32
  double* dd = scal + 32;                                          // diagonal of T (tail starts here)
  double* ed = dd + s;                                             // off-diagonal of T
  double* dn = ed + s;                                             // normalised diagonal
  double* e2n = dn + (s + 4);                                      // normalised off-diagonal^2
  double* bet = e2n + (s + 4);                                     // reflector scalars
  double* vv = bet + s;                                            // current reflector
  double* yy = vv + s;                                             // symv result
  double* ww = yy + s;                                             // (spare)
  double* lu = ww + s;                                             // nb * 4s
  unsigned char* piv = reinterpret_cast<unsigned char*>(lu + (size_t)nb * 4 * s);
  double* Ysub = dd;                                               // s x r (subspace iteration, aliases the tail)
  double* Hs = Ysub + s * r;                                       // r x r
  double* Cs = Hs + r * r;                                         // r x r
  double* Rs = Cs + r * r;                                         // r x r
  (void)ww;

  double* cred = lu;                                               // cluster partials: 3 x 16 EIG_CLUSTER
  long long* tm = ea.tmark ? ea.tmark + 8 * mi : nullptr;
  if (crank != 0) tm = nullptr;
  if (tm && tid == 0) tm[0] = clock64();
  const double* Kg = ea.K[mi];
  // (cluster helper CTAs, crank != 0, skip the load and the warm path: they wait at
  // S0 for CTA 0's verdict and join the tridiagonalisation below)
  if (crank == 0) {
  if (full) {
    for (int idx = tid; idx < npk; idx += blockDim.x) {
      int i = (int)((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
      while ((i + 1) * (i + 2) / 2 <= idx) ++i;
      while (i * (i + 1) / 2 > idx) --i;
      const int j = idx - i * (i + 1) / 2;
      const double v = Kg[idx];
      A[i * ld + j] = v;
      A[j * ld + i] = v;
    }
  } else {
    for (int i = tid; i < npk; i += blockDim.x) A[i] = Kg[i];
  }
  __syncthreads();
  if (tm && tid == 0) tm[1] = clock64();
  }

  // ---------------------------------------------------------------- 0. warm-started subspace iteration
  bool warm_ok = false;
  if (crank == 0 && ea.warmA[mi] != nullptr) {
    const bool ok = eig_subspace(A, full, ld, s, r, E, Ysub, Hs, Cs, Rs, red, red2, scal, ea.warmA[mi],
                                 ea.warm_rows[mi], ea.warm_d[mi], ea.max_sub_steps, tm);
    if (ok) {
      if (tid == 0 && ea.fast_used) ea.fast_used[mi] = (int)scal[14];   // subspace steps taken (>= 1)
      for (int e = tid; e < s * r; e += blockDim.x) ea.E[mi][e] = E[e];
      for (int j = tid; j < r; j += blockDim.x) ea.lam[mi][j] = 0.0;
      if (tm && tid == 0) tm[7] = clock64();
      warm_ok = true;
    }
  }
  // ---------------------------------------------------------------- 0b. Lanczos (full path, 64 <= s <= 256)
  // Lanczos with full (CGS2) reorthogonalisation from a fixed pseudo-random start
  // builds T_m = V_m^T K V_m; every 8 steps the r largest eigenpairs of T_m
  // (eig_tri_vectors: the same multisection + inverse iteration as the
  // Householder path, on the small T_m) give Ritz pairs with residuals
  // ||K V y - theta V y|| = beta_m |y_m|; once all r are below 1e-14 ||T_m|| the
  // Ritz vectors V_m Y are the eigenbasis (the Rayleigh-Ritz step of k_svdpost
  // then fixes the basis inside their span, as for the other paths).  The
  // Householder path needs s - 2 dependent steps; the top-r Ritz pairs of a
  // well separated spectrum converge in far fewer.  Full storage (s <= 128): K
  // stays in shared memory, the basis goes after the base layout.  Packed storage
  // (s > 128): the matvec reads the packed Gram from global memory (L2) and the
  // basis overwrites the shared-memory copy of K (the warm path is done with it).
  // Not converged within the basis capacity (or breakdown below r): the
  // Householder path below (K reloaded into shared memory when it was
  // overwritten).
  bool lz_done = false;
  if (!warm_ok && crank == 0 && ea.lz_mcap[mi] > 0) {
    if (tm && tid == 0) tm[2] = clock64();
    const int mcap = ea.lz_mcap[mi];
    double* V = full ? eig_smem + ea.lz_off[mi] : A;   // s x (mcap + 1), column k at V + k s
    double* hv = full ? V + (size_t)s * (mcap + 1) : yy;   // 2 (mcap + 1) projection coefficients (yy, ww adjacent)
    double* al = dd;                             // T_m diagonal
    double* be = ed;                             // T_m off-diagonal; be[m-1] = the residual norm
    double kn2 = 0.0;                            // ||K||_F^2 (breakdown scale)
    if (full) {
      for (int e = tid; e < s * s; e += blockDim.x) {
        const double v = A[(e / s) * ld + (e % s)];
        kn2 = fma(v, v, kn2);
      }
    } else {
      for (int i = wid; i < s; i += nw)
        for (int c = lane; c <= i; c += 32) {
          const double v = Kg[pk(i, c)];
          kn2 = fma(v, v * (c == i ? 1.0 : 2.0), kn2);
        }
    }
    __syncthreads();   // (packed: every thread is done reading K before the basis overwrites it)
    double v0 = 0.0;
    for (int i = tid; i < s; i += blockDim.x) {
      const double h = hash_unit(0x5DEECE66DULL ^ ((unsigned long long)i * 0x9E3779B9ULL));
      V[i] = h;
      v0 = fma(h, h, v0);
    }
    kn2 = warp_sum(kn2);
    v0 = warp_sum(v0);
    if (lane == 0) {
      red[wid] = kn2;
      red2[wid] = v0;
    }
    __syncthreads();
    const double knorm = sqrt(warp_sum_of(red, nw));
    const double vinv = 1.0 / sqrt(warp_sum_of(red2, nw));
    __syncthreads();
    for (int i = tid; i < s; i += blockDim.x) V[i] *= vinv;
    __syncthreads();
    int m = 0;
    bool conv = false;
    const int first_chk = max(16, 3 * r);
    for (int j = 0; j < mcap && !conv; ++j) {
      const double* vj = V + (size_t)j * s;
      double* w = V + (size_t)(j + 1) * s;
      // w = K v_j: rows by groups of EIG_TPR threads (128 groups; packed: K from L2)
      for (int ib = 0; ib < s; ib += (int)blockDim.x / EIG_TPR) {
        const int i = ib + tid / EIG_TPR, sub = tid & (EIG_TPR - 1);
        double acc = 0.0;
        if (i < s) {
          if (full) {
            const double* row = A + i * ld;
            double acc1 = 0.0;
            int c = sub;
            for (; c + EIG_TPR < s; c += 2 * EIG_TPR) {
              acc = fma(row[c], vj[c], acc);
              acc1 = fma(row[c + EIG_TPR], vj[c + EIG_TPR], acc1);
            }
            if (c < s) acc = fma(row[c], vj[c], acc);
            acc += acc1;
          } else if (ea.Kfull[mi]) {
            // row i of the mirrored copy: contiguous (the packed column part is a
            // strided walk, one sector per element)
            const double* row = ea.Kfull[mi] + (size_t)i * s;
            double acc1 = 0.0;
            int c = sub;
            for (; c + EIG_TPR < s; c += 2 * EIG_TPR) {
              acc = fma(__ldg(row + c), vj[c], acc);
              acc1 = fma(__ldg(row + c + EIG_TPR), vj[c + EIG_TPR], acc1);
            }
            if (c < s) acc = fma(__ldg(row + c), vj[c], acc);
            acc += acc1;
          } else {
            const double* row = Kg + pk(i, 0);
            for (int c = sub; c <= i; c += EIG_TPR) acc = fma(__ldg(row + c), vj[c], acc);
            int c = i + 1 + ((sub - (i + 1)) & (EIG_TPR - 1));
            for (; c < s; c += EIG_TPR) acc = fma(__ldg(Kg + pk(c, i)), vj[c], acc);
          }
        }
#pragma unroll
        for (int o = EIG_TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (i < s && sub == 0) w[i] = acc;
      }
      __syncthreads();
      // CGS2 against v_0..v_j; alpha_j = v_j^T K v_j from the two passes.  The
      // second pass also reduces ||w1||^2, so beta^2 = ||w1||^2 - ||h2||^2 (V
      // orthonormal) and the second update and the normalisation share one sweep;
      // under heavy cancellation (beta^2 < 0.01 ||w1||^2) beta is recomputed from
      // the updated vector instead.
      for (int k = wid; k <= j; k += nw) {
        const double* vk = V + (size_t)k * s;
        double d = 0.0;
        for (int t = lane; t < s; t += 32) d = fma(vk[t], w[t], d);
        d = warp_sum(d);
        if (lane == 0) hv[k] = d;
      }
      __syncthreads();
      if (tid == 0) al[j] = hv[j];
      for (int t = tid; t < s; t += blockDim.x) {
        double v = w[t];
        for (int k = 0; k <= j; ++k) v = fma(-hv[k], V[(size_t)k * s + t], v);
        w[t] = v;
      }
      __syncthreads();
      double* h2 = hv + (mcap + 1);   // (second-pass coefficients; hv has 2 (mcap + 1) doubles)
      for (int k = wid; k <= j; k += nw) {
        const double* vk = V + (size_t)k * s;
        double d = 0.0;
        for (int t = lane; t < s; t += 32) d = fma(vk[t], w[t], d);
        d = warp_sum(d);
        if (lane == 0) h2[k] = d;
      }
      {
        double nn = 0.0;
        for (int t = tid; t < s; t += blockDim.x) nn = fma(w[t], w[t], nn);
        nn = warp_sum(nn);
        if (lane == 0) red2[wid] = nn;
      }
      __syncthreads();
      if (tid == 0) al[j] += h2[j];
      const double n1 = warp_sum_of(red2, nw);
      double hh = 0.0;
      for (int k = 0; k <= j; ++k) hh = fma(h2[k], h2[k], hh);
      double b;
      if (n1 - hh >= 0.01 * n1) {
        b = sqrt(n1 - hh);
        const double bi = b > 0.0 ? 1.0 / b : 0.0;
        for (int t = tid; t < s; t += blockDim.x) {
          double v = w[t];
          for (int k = 0; k <= j; ++k) v = fma(-h2[k], V[(size_t)k * s + t], v);
          w[t] = v * bi;
        }
        __syncthreads();
      } else {
        for (int t = tid; t < s; t += blockDim.x) {
          double v = w[t];
          for (int k = 0; k <= j; ++k) v = fma(-h2[k], V[(size_t)k * s + t], v);
          w[t] = v;
        }
        __syncthreads();
        double nn = 0.0;
        for (int t = tid; t < s; t += blockDim.x) nn = fma(w[t], w[t], nn);
        nn = warp_sum(nn);
        if (lane == 0) red[wid] = nn;
        __syncthreads();
        b = sqrt(warp_sum_of(red, nw));
        const double bi = b > 0.0 ? 1.0 / b : 0.0;
        for (int t = tid; t < s; t += blockDim.x) w[t] *= bi;
        __syncthreads();
      }
      m = j + 1;
      const bool brk = !(b > 1e-13 * knorm);   // invariant subspace: T_m is exact
      if (tid == 0) be[j] = brk ? 0.0 : b;
      if (brk && m < r) break;   // fewer than r directions: the Householder path
      if (brk || m == mcap || (m >= first_chk && (m - first_chk) % ea.lz_stride == 0)) {
        if (tid == 0) eig_tri_bounds(al, be, m, scal);
        __syncthreads();
        const double tn = scal[0];
        if (tn > 0.0) {
          eig_tri_vectors(ea, mi, m, r, nb, tn, al, be, dn, e2n, lam, clus, red, red2, scal, lu, piv, E, nullptr);
          double rmax = 0.0;
          for (int c = 0; c < r; ++c) rmax = fmax(rmax, fabs(be[m - 1] * E[(size_t)c * m + m - 1]));
          conv = rmax <= 1e-14 * tn;   // (block-uniform: every thread reads the same values)
        }
        __syncthreads();
      }
    }
    if (conv) {
      // Ritz vectors V_m Y (s x r) straight to the output
      double* Eo = ea.E[mi];
      for (int e = tid; e < s * r; e += blockDim.x) {
        const int i = e % s, c = e / s;
        double acc = 0.0;
        for (int k = 0; k < m; ++k) acc = fma(V[(size_t)k * s + i], E[(size_t)c * m + k], acc);
        Eo[e] = acc;
      }
      if (tid == 0 && ea.fast_used) ea.fast_used[mi] = -m;   // (diagnostic: Lanczos steps, negated)
      if (tm && tid == 0) tm[3] = clock64();   // (eig_paths: span 2 = the Lanczos solve)
      lz_done = true;
    } else if (!full) {
      __syncthreads();   // the basis overwrote the packed K: reload it for the Householder path
      for (int i = tid; i < npk; i += blockDim.x) A[i] = Kg[i];
    }
    __syncthreads();
  }

  warm_ok |= lz_done;
  if (use_cl) {   // tell the helper CTAs whether the full path runs (scal[20] of every CTA)
    __syncthreads();
    if (crank == 0 && tid == 0)
      for (int c2 = 0; c2 < EIG_CLUSTER; ++c2) eig_put<EIG_CLUSTER>(scal + 20, c2, warm_ok ? 1.0 : 0.0);
    cg::this_cluster().sync();                                     // S0
    warm_ok = scal[20] != 0.0;
  }
  if (warm_ok) return;   // (warm path or Lanczos)
  if (crank == 0 && tid == 0 && ea.fast_used) ea.fast_used[mi] = 0;

  // ---------------------------------------------------------------- 1. tridiagonalise
  int hoff = 0;
  // register-tiled paths: clusters for 128 < s <= 256, single CTA for s <= 128 (RTCUR_EIG_REG=2)
  const bool regtri = (full && s >= 3 && s <= 128 && ea.reg_tridiag >= 2) || use_cl;
  if (use_cl) {
    // reflectors go contiguous into the (consumed) packed matrix area
    HV = A;
    hoff = eig_tridiag_reg<EIG_CLUSTER, 2, 8>(nullptr, 0, Kg, s, HV, dd, ed, bet, vv, ww, yy, cred,
                                              cred + 2 * 16 * EIG_CLUSTER);
    if (crank != 0) return;   // helpers are done; CTA 0 goes on alone
  } else if (regtri) {
    if (s <= 64) hoff = eig_tridiag_reg<1, 4, 2>(A, ld, nullptr, s, HV, dd, ed, bet, vv, ww, yy, red, red2);
    else hoff = eig_tridiag_reg<1, 8, 4>(A, ld, nullptr, s, HV, dd, ed, bet, vv, ww, yy, red, red2);
  } else if (full) {
    // Full symmetric storage.  The column k+1 that step k+1 reflects is produced
    // by step k's rank-2 update (row groups own it), so its squared norm is
    // reduced there: 2 barriers per Householder step.
    double* vbuf0 = vv;
    double* vbuf1 = ww;
    {
      const int L = s - 1;
      double sq = 0.0;
      for (int i = tid; i < L; i += blockDim.x) {
        const double x = A[(1 + i) * ld];
        vbuf0[i] = x;
        sq = fma(x, x, sq);
      }
      sq = warp_sum(sq);
      if (lane == 0) red[wid] = sq;
    }
    __syncthreads();
    const int sub = tid & (EIG_TPR - 1);
    const int gpw = 32 / EIG_TPR;          // row groups per warp
    for (int k = 0; k + 2 < s; ++k) {
      const int L = s - k - 1, b0 = k + 1;
      double* vc = (k & 1) ? vbuf1 : vbuf0;   // this step's column / reflector
      double* vn = (k & 1) ? vbuf0 : vbuf1;   // next step's column
      double* rc = (k & 1) ? red + 16 : red;  // this step's column norm partials (<= 16 warps)
      double* rn = (k & 1) ? red : red + 16;
      const double nrm = sqrt(warp_sum_of(rc, nw));
      const double x0 = vc[0];
      double alpha = 0.0, beta = 0.0;
      if (nrm > 0.0) {
        alpha = -copysign(nrm, x0);
        beta = 1.0 / (nrm * (nrm + fabs(x0)));
      }
      const double v0 = x0 - alpha;
      // y = beta * A22 v: row groups of EIG_TPR threads (warp-uniform trip count)
      double dotp = 0.0;
      for (int ib = wid * gpw; ib < L; ib += nw * gpw) {
        const int i = ib + lane / EIG_TPR;
        double a0 = 0.0, a1 = 0.0;
        if (i < L) {
          const double* __restrict__ row = A + (b0 + i) * ld + b0;
          int j = sub;
          if (sub == 0) { a0 = row[0] * v0; j = EIG_TPR; }
          for (; j + 3 * EIG_TPR < L; j += 4 * EIG_TPR) {
            double rv[4], vv4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { rv[u] = row[j + u * EIG_TPR]; vv4[u] = vc[j + u * EIG_TPR]; }
            a0 = fma(rv[0], vv4[0], a0);
            a1 = fma(rv[1], vv4[1], a1);
            a0 = fma(rv[2], vv4[2], a0);
            a1 = fma(rv[3], vv4[3], a1);
          }
          for (; j < L; j += EIG_TPR) a0 = fma(row[j], vc[j], a0);
        }
        double acc = a0 + a1;
#pragma unroll
        for (int o = EIG_TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        acc *= beta;
        if (i < L && sub == 0) {
          yy[i] = acc;
          dotp = fma(acc, i == 0 ? v0 : vc[i], dotp);
        }
      }
      dotp = warp_sum(dotp);
      if (lane == 0) red2[wid] = dotp;
      __syncthreads();                                             // B1
      const double kk = 0.5 * beta * warp_sum_of(red2, nw);
      // A22 -= v w^T + w v^T (w = y - kk v); the new column k+1 (local column 0,
      // rows >= 1) goes to vn with its squared norm
      double sq = 0.0;
      for (int ib = wid * gpw; ib < L; ib += nw * gpw) {
        const int i = ib + lane / EIG_TPR;
        if (i < L) {
          const double vi = i == 0 ? v0 : vc[i];
          const double wi = yy[i] - kk * vi;
          double* __restrict__ row = A + (b0 + i) * ld + b0;
          if (sub == 0) {
            // column 0 (next step's reflector input) first
            const double nv = row[0] - (vi * (yy[0] - kk * v0) + wi * v0);
            row[0] = nv;
            if (i >= 1) {
              vn[i - 1] = nv;
              sq = fma(nv, nv, sq);
            }
          }
          int j = (sub == 0) ? EIG_TPR : sub;
          for (; j + 3 * EIG_TPR < L; j += 4 * EIG_TPR) {
            double rv[4], vv4[4], yv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              rv[u] = row[j + u * EIG_TPR];
              vv4[u] = vc[j + u * EIG_TPR];
              yv[u] = yy[j + u * EIG_TPR];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) row[j + u * EIG_TPR] = rv[u] - (vi * (yv[u] - kk * vv4[u]) + wi * vv4[u]);
          }
          for (; j < L; j += EIG_TPR) {
            const double vj = vc[j];
            row[j] -= vi * (yy[j] - kk * vj) + wi * vj;
          }
        }
      }
      sq = warp_sum(sq);
      if (lane == 0) rn[wid] = sq;
      for (int i = tid; i < L; i += blockDim.x) HV[hoff + i] = i == 0 ? v0 : vc[i];
      if (tid == 0) {
        dd[k] = A[k * ld + k];
        ed[k] = alpha;
        bet[k] = beta;
      }
      hoff += L;
      __syncthreads();                                             // B2
    }
  } else {
    // Packed lower storage.  Matvec by row groups of EIG_TPR threads: row part
    // j <= i contiguous in the packed row, column part j > i read as column i of
    // rows j (consecutive rows of a warp hit consecutive words).  The rank-2
    // update touches the lower triangle only, each row group taking the row pair
    // (g, L-1-g) for balance, and produces the next column (+ its norm): 2 barriers
    // per Householder step.
    double* vbuf0 = vv;
    double* vbuf1 = ww;
    {
      double sq = 0.0;
      for (int i = tid; i < s - 1; i += blockDim.x) {
        const double x = A[pk(1 + i, 0)];
        vbuf0[i] = x;
        sq = fma(x, x, sq);
      }
      sq = warp_sum(sq);
      if (lane == 0) red[wid] = sq;
    }
    __syncthreads();
    const int sub = tid & (EIG_TPR - 1);
    const int grp = tid / EIG_TPR, ngrp = blockDim.x / EIG_TPR;
    const int gpw = 32 / EIG_TPR;
    for (int k = 0; k + 2 < s; ++k) {
      const int L = s - k - 1, b0 = k + 1;
      double* vc = (k & 1) ? vbuf1 : vbuf0;
      double* vn = (k & 1) ? vbuf0 : vbuf1;
      double* rc = (k & 1) ? red + 16 : red;
      double* rn = (k & 1) ? red : red + 16;
      const double nrm = sqrt(warp_sum_of(rc, nw));
      const double x0 = vc[0];
      double alpha = 0.0, beta = 0.0;
      if (nrm > 0.0) {
        alpha = -copysign(nrm, x0);
        beta = 1.0 / (nrm * (nrm + fabs(x0)));
      }
      const double v0 = x0 - alpha;
      // y = beta * A22 v
      double dotp = 0.0;
      for (int ib = wid * gpw; ib < L; ib += nw * gpw) {
        const int i = ib + lane / EIG_TPR;
        double a0 = 0.0, a1 = 0.0;
        if (i < L) {
          const int gi = b0 + i;
          const double* __restrict__ row = A + pk(gi, b0);
          int j = sub;
          if (sub == 0) { a0 = row[0] * v0; j = EIG_TPR; }
          for (; j <= i; j += EIG_TPR) a0 = fma(row[j], vc[j], a0);
          // first column-part index >= i+1 with j = sub (mod EIG_TPR)
          j = i + 1 + ((sub - (i + 1)) & (EIG_TPR - 1));
          int cb = pk(b0 + j, gi);
          for (; j < L; j += EIG_TPR) {
            a1 = fma(A[cb], vc[j], a1);
            cb += EIG_TPR * (b0 + j) + (EIG_TPR * (EIG_TPR + 1)) / 2;
          }
        }
        double acc = a0 + a1;
#pragma unroll
        for (int o = EIG_TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        acc *= beta;
        if (i < L && sub == 0) {
          yy[i] = acc;
          dotp = fma(acc, i == 0 ? v0 : vc[i], dotp);
        }
      }
      dotp = warp_sum(dotp);
      if (lane == 0) red2[wid] = dotp;
      __syncthreads();                                             // B1
      const double kk = 0.5 * beta * warp_sum_of(red2, nw);
      const double w0 = yy[0] - kk * v0;
      double sq = 0.0;
      for (int g = grp; g < (L + 1) / 2; g += ngrp) {
        for (int pass = 0; pass < 2; ++pass) {
          const int i = pass == 0 ? g : L - 1 - g;
          if (pass == 1 && i == g) break;
          const int gi = b0 + i;
          const double vi = i == 0 ? v0 : vc[i];
          const double wi = yy[i] - kk * vi;
          double* __restrict__ row = A + pk(gi, b0);
          int j = sub;
          if (sub == 0) {
            // column b0 (the next step's reflector input) first
            const double nv = row[0] - (vi * w0 + wi * v0);
            row[0] = nv;
            if (i >= 1) {
              vn[i - 1] = nv;
              sq = fma(nv, nv, sq);
            }
            A[pk(gi, k)] = vi;   // reflector in place (column k left the active block)
            j = EIG_TPR;
          }
          for (; j <= i; j += EIG_TPR) {
            const double vj = vc[j];
            row[j] -= vi * (yy[j] - kk * vj) + wi * vj;
          }
        }
      }
      sq = warp_sum(sq);
      if (lane == 0) rn[wid] = sq;
      if (tid == 0) {
        dd[k] = A[pk(k, k)];
        ed[k] = alpha;
        bet[k] = beta;
      }
      hoff += L;
      __syncthreads();                                             // B2
    }
  }
  if (tid == 0) {
    if (!regtri) {   // (the register path wrote the trailing 2x2 block itself)
      if (s >= 2) {
        dd[s - 2] = full ? A[(s - 2) * ld + s - 2] : A[pk(s - 2, s - 2)];
        ed[s - 2] = full ? A[(s - 1) * ld + s - 2] : A[pk(s - 1, s - 2)];
      }
      dd[s - 1] = full ? A[(s - 1) * ld + s - 1] : A[pk(s - 1, s - 1)];
    }
    eig_tri_bounds(dd, ed, s, scal);
  }
  __syncthreads();
  if (tm && tid == 0) tm[2] = clock64();
  const double tn = scal[0];
  double* Eout = ea.E[mi];

  if (tn == 0.0) {
    // zero matrix: every eigenvalue is 0, any orthonormal basis is exact
    for (int e = tid; e < s * r; e += blockDim.x) Eout[e] = (e % s == e / s) ? 1.0 : 0.0;
    for (int j = tid; j < r; j += blockDim.x) ea.lam[mi][j] = 0.0;
    return;
  }

  eig_tri_vectors(ea, mi, s, r, nb, tn, dd, ed, dn, e2n, lam, clus, red, red2, scal, lu, piv, E, tm);

  // ---------------------------------------------------------------- 4. back-transform
  for (int j = wid; j < r; j += nw) {
    double* x = E + j * s;
    int off = hoff;
    for (int k = s - 3; k >= 0; --k) {
      const int L = s - k - 1;
      off -= L;
      const double beta = bet[k];
      if (beta == 0.0) continue;
      double d = 0.0;
      if (full || regtri) {
        const double* v = HV + off;
        for (int i = lane; i < L; i += 32) d = fma(v[i], x[k + 1 + i], d);
        d = warp_sum(d) * beta;
        for (int i = lane; i < L; i += 32) x[k + 1 + i] = fma(-d, v[i], x[k + 1 + i]);
      } else {
        for (int i = lane; i < L; i += 32) d = fma(A[pk(k + 1 + i, k)], x[k + 1 + i], d);
        d = warp_sum(d) * beta;
        for (int i = lane; i < L; i += 32) x[k + 1 + i] = fma(-d, A[pk(k + 1 + i, k)], x[k + 1 + i]);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (tm && tid == 0) tm[5] = clock64();
  for (int e = tid; e < s * r; e += blockDim.x) Eout[e] = E[e];
}
