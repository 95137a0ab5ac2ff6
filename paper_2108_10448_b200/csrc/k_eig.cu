// k_eig.cu -- top-r eigenvectors of a small symmetric PSD matrix (the
// intersection Gram, s <= 235), one CTA per matrix, fp64 throughout:
//
//   1. Householder tridiagonalisation K = Q T Q^T, packed lower K in shared
//      memory (warp-per-row symv and rank-2 update; reflectors go to global).
//   2. The r largest eigenvalues of T by multisection on Sturm counts (each
//      warp owns one eigenvalue; 32 lanes test 32 shifts per round,
//      division-free three-term recurrence with exact power-of-2 rescaling).
//   3. Block inverse iteration on T (thread-per-vector pivoted tridiagonal LU,
//      3 solves) with block classical Gram-Schmidt (twice) after each solve,
//      so clusters converge to their invariant subspace.
//   4. Back-transform by the stored reflectors (warp-per-vector, no barriers).
//
// Only the span of the r vectors must be accurate: the Rayleigh-Ritz step in
// k_svdpost.cu fixes the basis inside it and recomputes the singular values
// from the intersection itself.  Replaces the dense_svd call of
// linalg.py:73 (_core.pyx:24-249) for the rank-r part the solver uses.
#include "common.cuh"
#include <cfloat>

struct EigArgs {
  int n;
  int s[RT_MAX_MODES];
  int r[RT_MAX_MODES];
  const double* K[RT_MAX_MODES];   // packed lower, s(s+1)/2
  double* hv[RT_MAX_MODES];        // reflectors: s*(s-1)/2 + s doubles
  double* E[RT_MAX_MODES];         // s x r, column-major (output)
  double* lam[RT_MAX_MODES];       // r, descending (output)
  int nb[RT_MAX_MODES];            // inverse-iteration batch (vectors factored at once)
};

__device__ __forceinline__ i64 pk(int i, int j) { return (i64)i * (i + 1) / 2 + j; }  // i >= j

__device__ __forceinline__ double hash_unit(unsigned long long a) {
  a += 0x9E3779B97F4A7C15ull;
  a = (a ^ (a >> 30)) * 0xBF58476D1CE4E5B9ull;
  a = (a ^ (a >> 27)) * 0x94D049BB133111EBull;
  a ^= a >> 31;
  return (double)(a >> 11) * (2.0 / 9007199254740992.0) - 1.0;   // (-1, 1)
}

// number of eigenvalues of T (dd, ed) strictly less than x
__device__ int sturm_count(const double* dd, const double* ed, int s, double x, double pivmin) {
  double pm2 = 1.0, pm1 = dd[0] - x;
  int cnt = 0;
  double sp = 1.0;
  if (pm1 == 0.0) pm1 = -pivmin;
  if ((pm1 < 0.0) != (sp < 0.0)) ++cnt;
  sp = pm1;
  for (int i = 1; i < s; ++i) {
    const double e = ed[i - 1];
    double p = (dd[i] - x) * pm1 - (e * e) * pm2;
    if (p == 0.0) p = -pivmin * pm1;
    if ((p < 0.0) != (sp < 0.0)) ++cnt;
    sp = p;
    const double ap = fabs(p);
    if (ap > 0x1p+400 || ap < 0x1p-400) {
      const int ex = ilogb(p);
      pm1 = ldexp(pm1, -ex);
      p = ldexp(p, -ex);
    }
    pm2 = pm1;
    pm1 = p;
  }
  return cnt;
}

extern __shared__ double eig_smem[];

__global__ void __launch_bounds__(1024) k_eig(EigArgs ea) {
  const int mi = blockIdx.x;
  if (mi >= ea.n) return;
  const int s = ea.s[mi], r = ea.r[mi];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const i64 npk = (i64)s * (s + 1) / 2;
  const int nb = ea.nb[mi];
  const i64 region0 = max(npk, (i64)5 * s * nb);
  double* A = eig_smem;
  double* dd = eig_smem + region0;
  double* ed = dd + s;
  double* vv = ed + s;
  double* yy = vv + s;
  double* ww = yy + s;
  double* red = ww + s;     // 32
  __shared__ double sh_beta, sh_tn, sh_lo, sh_hi;
  double* hv = ea.hv[mi];
  double* hb = hv + (i64)s * (s - 1) / 2;   // betas
  double* E = ea.E[mi];

  for (i64 i = tid; i < npk; i += blockDim.x) A[i] = ea.K[mi][i];
  __syncthreads();

  // ---------------------------------------------------------------- 1. tridiagonalise
  i64 hoff = 0;
  for (int k = 0; k + 2 < s; ++k) {
    const int L = s - k - 1;
    double sq = 0.0;
    for (int i = tid; i < L; i += blockDim.x) {
      const double x = A[pk(k + 1 + i, k)];
      vv[i] = x;
      sq = fma(x, x, sq);
    }
    sq = block_sum(sq, red);
    if (tid == 0) {
      const double x0 = vv[0];
      const double nrm = sqrt(sq);
      dd[k] = A[pk(k, k)];
      if (nrm == 0.0) {
        sh_beta = 0.0;
        ed[k] = 0.0;
      } else {
        const double alpha = -copysign(nrm, x0);
        vv[0] = x0 - alpha;
        sh_beta = 1.0 / (nrm * (nrm + fabs(x0)));
        ed[k] = alpha;
      }
      hb[k] = sh_beta;
    }
    __syncthreads();
    const double beta = sh_beta;
    for (int i = tid; i < L; i += blockDim.x) hv[hoff + i] = vv[i];
    if (beta != 0.0) {
      // y = beta * A22 v   (warp per row; A22[i][j] = A[k+1+max, k+1+min])
      for (int i = wid; i < L; i += nw) {
        const int gi = k + 1 + i;
        double acc = 0.0;
        const i64 rowbase = pk(gi, k + 1);
        for (int j = lane; j < L; j += 32) {
          const double a = (j <= i) ? A[rowbase + j] : A[pk(k + 1 + j, gi)];
          acc = fma(a, vv[j], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) yy[i] = beta * acc;
      }
      __syncthreads();
      double dot = 0.0;
      for (int i = tid; i < L; i += blockDim.x) dot = fma(yy[i], vv[i], dot);
      dot = block_sum(dot, red);
      const double kk = 0.5 * beta * dot;
      for (int i = tid; i < L; i += blockDim.x) ww[i] = yy[i] - kk * vv[i];
      __syncthreads();
      for (int i = wid; i < L; i += nw) {
        const double vi = vv[i], wi = ww[i];
        const i64 rowbase = pk(k + 1 + i, k + 1);
        for (int j = lane; j <= i; j += 32) A[rowbase + j] -= vi * ww[j] + wi * vv[j];
      }
    }
    __syncthreads();
    hoff += L;
  }
  if (tid == 0) {
    if (s >= 2) {
      dd[s - 2] = A[pk(s - 2, s - 2)];
      ed[s - 2] = A[pk(s - 1, s - 2)];
    }
    dd[s - 1] = A[pk(s - 1, s - 1)];
    double tn = 0.0, lo = DBL_MAX, hi = -DBL_MAX;
    for (int i = 0; i < s; ++i) {
      const double rad = (i > 0 ? fabs(ed[i - 1]) : 0.0) + (i + 1 < s ? fabs(ed[i]) : 0.0);
      tn = fmax(tn, fabs(dd[i]) + rad);
      lo = fmin(lo, dd[i] - rad);
      hi = fmax(hi, dd[i] + rad);
    }
    sh_tn = tn;
    sh_lo = lo;
    sh_hi = hi;
  }
  __syncthreads();
  const double tn = sh_tn;

  if (tn == 0.0) {
    // zero matrix: every eigenvalue is 0, any orthonormal basis is exact
    for (int j = 0; j < r; ++j) {
      for (int i = tid; i < s; i += blockDim.x) E[i + (i64)j * s] = (i == j) ? 1.0 : 0.0;
      if (tid == 0) ea.lam[mi][j] = 0.0;
    }
    return;
  }

  // ---------------------------------------------------------------- 2. multisection
  const double pivmin = DBL_MIN * fmax(1.0, tn * tn);
  const double pad = 2.0 * DBL_EPSILON * tn * s + pivmin;
  double* lam = yy;   // reuse (s >= r)
  for (int j = wid; j < r; j += nw) {
    const int target = s - 1 - j;   // ascending index of the j-th largest
    double lo = sh_lo - pad, hi = sh_hi + pad;
    for (int round = 0; round < 24; ++round) {
      const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
      const int c = sturm_count(dd, ed, s, x, pivmin);
      double nlo = (c <= target) ? x : -DBL_MAX;
      double nhi = (c >= target + 1) ? x : DBL_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        nlo = fmax(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
        nhi = fmin(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
      }
      if (nlo != -DBL_MAX) lo = nlo;
      if (nhi != DBL_MAX) hi = nhi;
      if (lo >= hi) { const double mid = 0.5 * (lo + hi); lo = hi = mid; break; }
      if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin || hi - lo <= 0.25 * DBL_EPSILON * tn) break;
    }
    if (lane == 0) lam[j] = 0.5 * (lo + hi);
  }
  __syncthreads();
  for (int j = tid; j < r; j += blockDim.x) ea.lam[mi][j] = lam[j];

  // ---------------------------------------------------------------- 3. block inverse iteration
  const double tiny = DBL_EPSILON * tn;
  const double pertol = 10.0 * DBL_EPSILON * tn;
  for (int j0 = 0; j0 < r; j0 += nb) {
    const int jn = min(nb, r - j0);
    // thread t < jn owns vector j0+t: factor T - mu I with partial pivoting
    double* u0 = A + (i64)5 * s * tid;
    double* u1 = u0 + s;
    double* u2 = u1 + s;
    double* lm = u2 + s;
    double* pv = lm + s;
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
        double l;
        if (fabs(ca) >= fabs(c)) {
          if (fabs(ca) < tiny) ca = copysign(tiny, ca);
          l = c / ca;
          u0[i] = 1.0 / ca;
          u1[i] = cb;
          u2[i] = 0.0;
          pv[i] = 0.0;
          ca = na - l * cb;
          cb = nbv;
        } else {
          l = ca / c;
          u0[i] = 1.0 / c;
          u1[i] = na;
          u2[i] = nbv;
          pv[i] = 1.0;
          ca = cb - l * na;
          cb = -l * nbv;
        }
        lm[i] = l;
      }
      if (fabs(ca) < tiny) ca = copysign(tiny, ca);
      u0[s - 1] = 1.0 / ca;
      double* x = E + (i64)j * s;
      for (int i = 0; i < s; ++i) x[i] = hash_unit(((unsigned long long)j << 32) ^ (unsigned long long)i);
    }
    __syncthreads();
    for (int it = 0; it < 3; ++it) {
      if (tid < jn) {
        double* x = E + (i64)(j0 + tid) * s;
        // forward: apply P and L^-1
        for (int i = 0; i + 1 < s; ++i) {
          double bi = x[i], bn = x[i + 1];
          if (pv[i] != 0.0) { const double t = bi; bi = bn; bn = t; x[i] = bi; }
          x[i + 1] = bn - lm[i] * bi;
        }
        // back substitution with U (diag reciprocal u0, supers u1, u2)
        double xn1 = 0.0, xn2 = 0.0;
        for (int i = s - 1; i >= 0; --i) {
          double v = x[i];
          if (i + 1 < s) v -= u1[i] * xn1;
          if (i + 2 < s) v -= u2[i] * xn2;
          v *= u0[i];
          if (!isfinite(v)) v = 0.0;
          x[i] = v;
          xn2 = xn1;
          xn1 = v;
        }
        // scale to unit max so the next solve cannot overflow
        double mx = 0.0;
        for (int i = 0; i < s; ++i) mx = fmax(mx, fabs(x[i]));
        if (mx > 0.0) {
          const double inv = 1.0 / mx;
          for (int i = 0; i < s; ++i) x[i] *= inv;
        }
      }
      __syncthreads();
      __threadfence_block();
      // block CGS2 over vectors 0..j0+jn-1 (earlier batches are final)
      for (int j = j0; j < j0 + jn; ++j) {
        double* xj = E + (i64)j * s;
        for (int pass = 0; pass < 2; ++pass) {
          // dots with all previous vectors: warp w handles vector i = w, w+nw, ...
          for (int i = wid; i < j; i += nw) {
            const double* xi = E + (i64)i * s;
            double d = 0.0;
            for (int t = lane; t < s; t += 32) d = fma(xi[t], xj[t], d);
            d = warp_sum(d);
            if (lane == 0) red[i % 32] = d;   // j <= 32 guaranteed by RT_MAX_RANK
          }
          __syncthreads();
          for (int t = tid; t < s; t += blockDim.x) {
            double v = xj[t];
            for (int i = 0; i < j; ++i) v = fma(-red[i], E[t + (i64)i * s], v);
            xj[t] = v;
          }
          __syncthreads();
        }
        double nn = 0.0;
        for (int t = tid; t < s; t += blockDim.x) nn = fma(xj[t], xj[t], nn);
        nn = block_sum(nn, red);
        if (nn > 0.0) {
          const double inv = 1.0 / sqrt(nn);
          for (int t = tid; t < s; t += blockDim.x) xj[t] *= inv;
        } else {
          // degenerate: replace with a unit vector, orthogonalised on the next pass
          for (int t = tid; t < s; t += blockDim.x) xj[t] = (t == j % s) ? 1.0 : 0.0;
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- 4. back-transform
  for (int j = wid; j < r; j += nw) {
    double* x = E + (i64)j * s;
    i64 off = hoff;
    for (int k = s - 3; k >= 0; --k) {
      const int L = s - k - 1;
      off -= L;
      const double beta = hb[k];
      if (beta == 0.0) continue;
      const double* v = hv + off;
      double d = 0.0;
      for (int i = lane; i < L; i += 32) d = fma(v[i], x[k + 1 + i], d);
      d = warp_sum(d) * beta;
      for (int i = lane; i < L; i += 32) x[k + 1 + i] -= d * v[i];
      __syncwarp();
    }
  }
}
