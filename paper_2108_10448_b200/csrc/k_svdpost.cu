// k_svdpost.cu -- finish the rank-r truncated SVD of each intersection from
// the short-side eigenbasis E (k_eig.cu):
//
//   Z  = B^T E            long-side projections (l x r)         k_zproj
//   H  = Z^T Z            r x r (split over l, deterministic)    k_hgram
//   H = Q diag(mu) Q^T    Rayleigh-Ritz rotation (warp Jacobi)   k_svd_fin1
//   S_short = E Q,  Z <- Z Q                                     k_zrot
//   H' = Z^T Z; sigma_a = sqrt(H'_aa) = ||z_a||, stable sort,
//   Cholesky of the normalised H' -> T with Z T orthonormal      k_svd_fin2
//   S_long = Z T (+ orthonormal completion for sigma <= tau)     k_long, k_complete
//
// Output per mode (matching linalg.py:26-56 TruncatedSvd): U (|I| x r),
// singular values (non-increasing), V (|J| x r), the truncated-pinv
// reciprocals 1/sigma for sigma > tau = max(m, p) * sigma_1 * 1e-12 (else 0,
// linalg.py:54-55) and the rank-deficiency flag of solver.py:252-257.
// U/V are stored row-major (row index major, r contiguous values per row).
#include "common.cuh"
#include <cfloat>

struct SvdArgs {
  const int* stop;   // the engine's stop flag (iteration launches), or null
  int n;
  int s[RT_MAX_MODES];
  i64 l[RT_MAX_MODES];
  int r[RT_MAX_MODES];
  int tall[RT_MAX_MODES];
  i64 mrows[RT_MAX_MODES];           // |I_k| (rows of M)
  i64 pcols[RT_MAX_MODES];           // |J_k|
  const double* M[RT_MAX_MODES];     // m x p column-major intersection
  const double* E[RT_MAX_MODES];     // s x r column-major eigenbasis
  double* Z[RT_MAX_MODES];           // l x r row-major
  double* hpart[RT_MAX_MODES];       // [chunks][r*r]
  double* H[RT_MAX_MODES];           // r x r
  double* Q[RT_MAX_MODES];           // r x r (col-major) Ritz rotation, then T
  double* U[RT_MAX_MODES];           // m x r row-major (output)
  double* V[RT_MAX_MODES];           // p x r row-major (output)
  double* sig[RT_MAX_MODES];         // r (output)
  double* siginv[RT_MAX_MODES];      // r (output)
  int* perm[RT_MAX_MODES];           // r
  int* degen[RT_MAX_MODES];          // r flags + [r] = any
  int* flags;                        // n rank-deficiency flags (output)
  int hchunk;                        // long-side rows per CTA for k_hgram
};

__device__ __forceinline__ double svd_B(const SvdArgs& sa, int k, i64 c, i64 t) {
  // B is s x l: B = M (wide) or M^T (tall)
  const double* M = sa.M[k];
  return sa.tall[k] ? M[t + c * sa.mrows[k]] : M[c + t * sa.mrows[k]];
}

// Z[t, a] = sum_c B[c, t] E[c, a]: a CTA owns ZP_T long-side columns t; the
// s x ZP_T slab of B and E (s x r) are staged in shared memory; thread
// (tl, a) = (tid % ZP_T, tid / ZP_T) reduces over c.
#define ZP_T 32
#define ZP_LD (ZP_T + 1)   // padded slab row: the wide-case transpose store is conflict-free
template <int R>
__global__ void __launch_bounds__(32 * R) k_zproj(SvdArgs sa) {
  if (rt_stopped(sa.stop)) return;
  extern __shared__ double es[];
  const int k = blockIdx.y;
  if (k >= sa.n) return;
  const int s = sa.s[k], r = sa.r[k];
  const i64 l = sa.l[k];
  const i64 t0 = (i64)blockIdx.x * ZP_T;
  if (t0 >= l) return;
  const int nt = (int)min((i64)ZP_T, l - t0);
  double* bs = es + s * r;   // s x ZP_LD
  for (int i = threadIdx.x; i < s * r; i += blockDim.x) es[i] = sa.E[k][i];
  const double* M = sa.M[k];
  const i64 mr = sa.mrows[k];
  if (sa.tall[k]) {
    // B[c, t] = M[t + c*m]: t contiguous
    for (int i = threadIdx.x; i < s * ZP_T; i += blockDim.x) {
      const int tl = i % ZP_T, c = i / ZP_T;
      bs[c * ZP_LD + tl] = tl < nt ? M[t0 + tl + (i64)c * mr] : 0.0;
    }
  } else {
    // B[c, t] = M[c + t*m]: c contiguous
    for (int i = threadIdx.x; i < s * ZP_T; i += blockDim.x) {
      const int c = i % s, tl = i / s;
      bs[c * ZP_LD + tl] = tl < nt ? M[c + (t0 + tl) * mr] : 0.0;
    }
  }
  __syncthreads();
  const int tl = threadIdx.x % ZP_T, a = threadIdx.x / ZP_T;
  if (a >= r || tl >= nt) return;
  const double* ea = es + a * s;
  double z0 = 0.0, z1 = 0.0;
  int c = 0;
  for (; c + 1 < s; c += 2) {
    z0 = fma(ea[c], bs[c * ZP_LD + tl], z0);
    z1 = fma(ea[c + 1], bs[(c + 1) * ZP_LD + tl], z1);
  }
  if (c < s) z0 = fma(ea[c], bs[c * ZP_LD + tl], z0);
  sa.Z[k][(t0 + tl) * r + a] = z0 + z1;
}

// Z <- Z Q (in place, per long-side row)
template <int R>
__global__ void __launch_bounds__(256) k_zrot(SvdArgs sa) {
  if (rt_stopped(sa.stop)) return;
  __shared__ double qs[RT_MAX_RANK * RT_MAX_RANK];
  const int k = blockIdx.y;
  if (k >= sa.n) return;
  const int r = sa.r[k];
  const i64 l = sa.l[k];
  if ((i64)blockIdx.x * blockDim.x >= l) return;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) qs[i] = sa.Q[k][i];
  __syncthreads();
  const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= l) return;
  double* Z = sa.Z[k] + t * r;
  double z[R], o[R];
#pragma unroll
  for (int a = 0; a < R; ++a) { z[a] = a < r ? Z[a] : 0.0; o[a] = 0.0; }
#pragma unroll
  for (int b = 0; b < R; ++b)
#pragma unroll
    for (int a = 0; a < R; ++a)
      if (a < r && b < r) o[a] = fma(z[b], qs[b + a * r], o[a]);
#pragma unroll
  for (int a = 0; a < R; ++a)
    if (a < r) Z[a] = o[a];
}

// H = Z^T Z: CTA = (chunk of HG_CH long rows, mode).  The chunk of Z is staged
// in shared memory; thread (pair, slice) sums a strided slice of rows; slices
// are combined in fixed order; the last CTA of each mode combines the chunk
// partials the same way (deterministic).
#define HG_CH 128
// PH 1: H = Z^T Z of the projections; the last CTA of each mode then runs the
//       Rayleigh-Ritz rotation (svd_fin1_warp) and writes the short-side vectors.
// PH 2: each CTA first rotates its Z rows by Q (Z <- Z Q, written back), H' = Z^T Z;
//       the last CTA runs svd_fin2_warp (sigma, order, cutoff, flags, T).
// PH 3: PH 1 and then the fin2 step on H' = Q^T H Q with T' = Q T (one launch; the
//       long side is Z T' from the unrotated Z).
__device__ void svd_fin1_warp(const SvdArgs& sa, int k);
__device__ void svd_fin2_warp(const SvdArgs& sa, int k);
__device__ void svd_fin2_ritz_warp(const SvdArgs& sa, int k, double* scr);
__device__ void svd_short_vecs_cta(const SvdArgs& sa, int k, int t0, int stride);
template <int PH>
__global__ void __launch_bounds__(512) k_hgram(SvdArgs sa, unsigned int* counters) {
  if (rt_stopped(sa.stop)) return;
  extern __shared__ double hz[];   // HG_CH * r + blockDim
  __shared__ bool am_last;
  __shared__ double qs[RT_MAX_RANK * RT_MAX_RANK];
  const int k = blockIdx.y;
  if (k >= sa.n) return;
  const int r = sa.r[k];
  const i64 l = sa.l[k];
  const int nch = (int)((l + HG_CH - 1) / HG_CH);
  if ((int)blockIdx.x >= nch) return;
  const int npair = r * (r + 1) / 2;
  const int nsl = max(1, (int)blockDim.x / npair);
  const int tid = threadIdx.x;
  const int pair = tid % npair, sl = tid / npair;
  int a = 0, b = 0;
  {
    int rem = pair;
    while (rem >= r - a) { rem -= r - a; ++a; }
    b = a + rem;
  }
  double* red = hz + HG_CH * r;
  const i64 t0 = (i64)blockIdx.x * HG_CH;
  const int nt = (int)min((i64)HG_CH, l - t0);
  double* Z = sa.Z[k] + t0 * r;
  if (PH == 2) {
    for (int i = tid; i < r * r; i += blockDim.x) qs[i] = sa.Q[k][i];
    __syncthreads();
    for (int t = tid; t < nt; t += blockDim.x) {   // Z <- Z Q, row t
      double z[RT_MAX_RANK];
      for (int b = 0; b < r; ++b) z[b] = Z[(i64)t * r + b];
      for (int a2 = 0; a2 < r; ++a2) {
        double o = 0.0;
        for (int b = 0; b < r; ++b) o = fma(z[b], qs[b + a2 * r], o);
        hz[t * r + a2] = o;
        Z[(i64)t * r + a2] = o;
      }
    }
  } else {
    for (int i = tid; i < nt * r; i += blockDim.x) hz[i] = Z[i];
  }
  __syncthreads();
  double acc = 0.0;
  if (sl < nsl)
    for (int t = sl; t < nt; t += nsl) acc = fma(hz[t * r + a], hz[t * r + b], acc);
  red[tid] = acc;
  __syncthreads();
  if (tid < npair) {
    double v = 0.0;
    for (int q = 0; q < nsl; ++q) v += red[q * npair + tid];
    sa.hpart[k][(i64)blockIdx.x * npair + tid] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = (atomicAdd(&counters[k], 1u) == (unsigned)nch - 1);
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  acc = 0.0;
  if (sl < nsl)
    for (int c = sl; c < nch; c += nsl) acc += ((volatile double*)sa.hpart[k])[(i64)c * npair + pair];
  red[tid] = acc;
  __syncthreads();
  if (tid < npair) {
    double v = 0.0;
    for (int q = 0; q < nsl; ++q) v += red[q * npair + tid];
    sa.H[k][a + b * r] = v;
    sa.H[k][b + a * r] = v;
  }
  if (tid == 0) counters[k] = 0u;
  __threadfence();
  __syncthreads();
  if (PH == 1 || PH == 3) {
    if (tid < 32) svd_fin1_warp(sa, k);
    __threadfence();
    __syncthreads();
    svd_short_vecs_cta(sa, k, tid, blockDim.x);
    if (PH == 3) {
      __syncthreads();   // (the short-side vectors have read Q)
      if (tid < 32) svd_fin2_ritz_warp(sa, k, hz);   // hz (the staged Z chunk) is free now
    }
  } else {
    if (tid < 32) svd_fin2_warp(sa, k);
  }
}

// Rayleigh-Ritz: cyclic Jacobi on H (one warp per mode, lane = row), sort the
// Ritz values descending, write Q (col-major) and the short-side vectors E Q.
// Rayleigh-Ritz rotation Q of mode k by one warp (lane = threadIdx.x & 31).
__device__ void svd_fin1_warp(const SvdArgs& sa, int k) {
  // Parallel (round-robin) Jacobi on the r x r symmetric H: each round rotates
  // the m/2 disjoint pairs of a tournament schedule at once (m = r rounded up
  // to even, index r is a bye), columns then rows, accumulating Q.
  __shared__ double h[RT_MAX_RANK * RT_MAX_RANK];
  __shared__ double q[RT_MAX_RANK * RT_MAX_RANK];
  __shared__ double rc[RT_MAX_RANK / 2 + 1], rs[RT_MAX_RANK / 2 + 1];
  __shared__ int pp[RT_MAX_RANK / 2 + 1], pq[RT_MAX_RANK / 2 + 1];
  __shared__ int ord[RT_MAX_RANK];
  const int r = sa.r[k], lane = threadIdx.x & 31;
  const int m = r + (r & 1), half = m / 2;
  for (int i = lane; i < r * r; i += 32) {
    h[i] = sa.H[k][i];
    q[i] = (i % r == i / r) ? 1.0 : 0.0;
  }
  __syncwarp();
  for (int sweep = 0; sweep < 40 && r > 1; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = lane; i < r * r; i += 32) {
      const double v = h[i] * h[i];
      if (i % r == i / r) dia += v; else off += v;
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (off <= 1e-30 * dia || off == 0.0) break;
    for (int round = 0; round < m - 1; ++round) {
      // tournament pairing: player 0 fixed, players 1..m-1 rotate by `round`
      if (lane < half) {
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (m - 1); };
        int a = player(lane), b = player(m - 1 - lane);
        if (a > b) { const int t = a; a = b; b = t; }
        double c = 1.0, sn = 0.0;
        if (b < r) {
          const double apq = h[a + b * r];
          if (apq != 0.0) {
            const double app = h[a + a * r], aqq = h[b + b * r];
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            sn = t * c;
          }
        }
        pp[lane] = a;
        pq[lane] = b;
        rc[lane] = c;
        rs[lane] = sn;
      }
      __syncwarp();
      // two-sided update in one pass: lane task = the 2x2 block (rows of pair u,
      // columns of pair w), column rotation first, then the row rotation -- the
      // same expressions in the same order as a column pass followed by a row pass
      for (int e = lane; e < half * half; e += 32) {
        const int u = e % half, w = e / half;
        const int pu = pp[u], qu = pq[u], pw = pp[w], qw = pq[w];
        const bool ru = qu < r, rw = qw < r;
        const double cu = rc[u], su = rs[u], cw = rc[w], sw = rs[w];
        double b00 = h[pu + pw * r], b01 = rw ? h[pu + qw * r] : 0.0;
        double b10 = ru ? h[qu + pw * r] : 0.0, b11 = (ru && rw) ? h[qu + qw * r] : 0.0;
        if (rw) {   // columns pw, qw
          const double t00 = cw * b00 - sw * b01, t01 = sw * b00 + cw * b01;
          const double t10 = cw * b10 - sw * b11, t11 = sw * b10 + cw * b11;
          b00 = t00; b01 = t01; b10 = t10; b11 = t11;
        }
        if (ru) {   // rows pu, qu
          const double t00 = cu * b00 - su * b10, t10 = su * b00 + cu * b10;
          const double t01 = cu * b01 - su * b11, t11 = su * b01 + cu * b11;
          b00 = t00; b01 = t01; b10 = t10; b11 = t11;
        }
        h[pu + pw * r] = b00;
        if (rw) h[pu + qw * r] = b01;
        if (ru) h[qu + pw * r] = b10;
        if (ru && rw) h[qu + qw * r] = b11;
      }
      // columns p, q of the accumulated rotation (lanes over (row, pair))
      for (int e = lane; e < r * half; e += 32) {
        const int row = e % r, pr = e / r;
        const int p = pp[pr], qq = pq[pr];
        if (qq >= r) continue;
        const double c = rc[pr], sn = rs[pr];
        const double qp = q[row + p * r], qv = q[row + qq * r];
        q[row + p * r] = c * qp - sn * qv;
        q[row + qq * r] = sn * qp + c * qv;
      }
      __syncwarp();
    }
  }
  if (lane == 0) {
    for (int i = 0; i < r; ++i) ord[i] = i;
    for (int i = 1; i < r; ++i) {
      const int t = ord[i];
      int j = i - 1;
      while (j >= 0 && h[ord[j] + ord[j] * r] < h[t + t * r]) { ord[j + 1] = ord[j]; --j; }
      ord[j + 1] = t;
    }
  }
  __syncwarp();
  for (int i = lane; i < r * r; i += 32) {
    const int row = i % r, col = i / r;
    sa.Q[k][i] = q[row + ord[col] * r];
  }
}

__global__ void __launch_bounds__(32) k_svd_fin1(SvdArgs sa) {
  if (rt_stopped(sa.stop)) return;
  if ((int)blockIdx.x < sa.n) svd_fin1_warp(sa, blockIdx.x);
}

// short-side vectors S = E Q written row-major into U (wide) or V (tall)
__device__ void svd_short_vecs_cta(const SvdArgs& sa, int k, int t0, int stride) {
  const int s = sa.s[k], r = sa.r[k];
  double* out = sa.tall[k] ? sa.V[k] : sa.U[k];
  for (int e = t0; e < s * r; e += stride) {
    const int i = e / r, a = e % r;
    double acc = 0.0;
    for (int b = 0; b < r; ++b) acc = fma(sa.E[k][i + b * s], sa.Q[k][b + a * r], acc);
    out[(i64)i * r + a] = acc;
  }
}
__global__ void k_short_vecs(SvdArgs sa) {
  if (rt_stopped(sa.stop)) return;
  const int k = blockIdx.y;
  if (k >= sa.n) return;
  svd_short_vecs_cta(sa, k, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// sigma from ||z_a||, stable descending order, truncated-pinv reciprocals,
// Cholesky orthonormalisation T (Z T orthonormal) over non-degenerate columns.
// scratch: 4 r^2 + r doubles and 2 r ints (shared memory)
// Stable descending order of v[0..r) by one warp: lane i's rank is the number of
// entries greater than v[i] plus the equal ones before it (the insertion sort's
// order); any NaN falls back to lane 0's insertion sort.
__device__ __forceinline__ void warp_order_desc(const double* v, int r, int* ord) {
  const int lane = threadIdx.x & 31;
  const bool nan = lane < r && isnan(v[lane]);
  if (__any_sync(0xffffffffu, nan)) {
    if (lane == 0) {
      for (int i = 0; i < r; ++i) ord[i] = i;
      for (int i = 1; i < r; ++i) {
        const int t = ord[i];
        int j = i - 1;
        while (j >= 0 && v[ord[j]] < v[t]) { ord[j + 1] = ord[j]; --j; }
        ord[j + 1] = t;
      }
    }
  } else if (lane < r) {
    const double x = v[lane];
    int rank = 0;
    for (int j = 0; j < r; ++j) rank += (v[j] > x) || (v[j] == x && j < lane);
    ord[rank] = lane;
  }
  __syncwarp();
}

// hsrc: H (r x r) in shared memory, or null to read sa.H.  The normalised
// Cholesky runs right-looking with lanes over columns: every entry sees the same
// subtractions in the same order (and the same divisions) as the column-by-column
// form, so the factor is bit-identical to it.  T is left in scratch + 2 r^2.
__device__ void svd_fin2_warp_s(const SvdArgs& sa, int k, double* scratch, const double* hsrc) {
  const int r = sa.r[k], lane = threadIdx.x & 31;
  double* h = scratch;
  double* R = h + r * r;
  double* T = R + r * r;
  double* X = T + r * r;
  double* sg = X + r * r;
  int* ord = reinterpret_cast<int*>(sg + r);
  int* dg = ord + r;
  const double* H = hsrc ? hsrc : sa.H[k];
  for (int i = lane; i < r * r; i += 32) {
    h[i] = H[i];
    R[i] = 0.0;
    T[i] = 0.0;
  }
  __syncwarp();
  if (lane < r) sg[lane] = sqrt(fmax(h[lane + lane * r], 0.0));
  __syncwarp();
  warp_order_desc(sg, r, ord);
  const double s1 = sg[ord[0]];
  const double mx = (double)(sa.mrows[k] > sa.pcols[k] ? sa.mrows[k] : sa.pcols[k]);
  const double tau = mx * s1 * 1e-12;   // linalg.py:54
  if (lane < r) {
    const double sv = sg[ord[lane]];
    sa.sig[k][lane] = sv;
    sa.siginv[k][lane] = sv > tau ? 1.0 / sv : 0.0;
    sa.perm[k][lane] = ord[lane];
    dg[lane] = !(sv > tau);
  }
  if (lane == 0) {
    // flags: solver.py:252-257 (sigma_1 <= 0 or sigma_r <= 1e-8 sigma_1)
    sa.flags[k] = (s1 <= 0.0 || sg[ord[r - 1]] <= 1e-8 * s1) ? 1 : 0;
  }
  __syncwarp();
  // Cholesky of C = D^-1 P^T H P D^-1 on the non-degenerate columns; X holds the
  // working upper triangle (lane j owns column j)
  if (lane < r) {
    const int oj = ord[lane];
    for (int i = 0; i <= lane; ++i) {
      const int oi = ord[i];
      X[i + lane * r] = h[oi + oj * r] / (sg[oi] * sg[oj]);
    }
  }
  __syncwarp();
  for (int p = 0; p < r; ++p) {
    if (dg[p]) continue;   // (warp-uniform) row p of R stays zero
    const double c = X[p + p * r];
    if (c <= 1e-6) {   // numerically dependent: complete instead
      __syncwarp();
      if (lane == 0) dg[p] = 1;
      __syncwarp();
      continue;
    }
    const double d = sqrt(c);
    if (lane == p) R[p + p * r] = d;
    if (lane > p && lane < r) R[p + lane * r] = X[p + lane * r] / d;
    __syncwarp();
    if (lane > p && lane < r) {
      const double rj = R[p + lane * r];
      for (int i = p + 1; i <= lane; ++i) X[i + lane * r] -= R[p + i * r] * rj;
    }
    __syncwarp();
  }
  // T = P D^-1 R^-1: lane j solves R x = e_j (upper triangular) for column j
  // (into column j of X: the working triangle is no longer needed)
  __syncwarp();
  if (lane < r && !dg[lane]) {
    const int j = lane;
    double* x = X + j * r;
    for (int i = j; i >= 0; --i) {
      if (dg[i]) { x[i] = 0.0; continue; }
      double v = (i == j) ? 1.0 : 0.0;
      for (int p = i + 1; p <= j; ++p)
        if (!dg[p]) v -= R[i + p * r] * x[p];
      x[i] = v / R[i + i * r];
    }
    for (int i = 0; i <= j; ++i)
      if (!dg[i]) T[ord[i] + j * r] = x[i] / sg[ord[i]];
  }
  __syncwarp();
  for (int i = lane; i < r * r; i += 32) sa.Q[k][i] = T[i];
  int anyd = 0;
  for (int a = 0; a < r; ++a) anyd |= dg[a];
  if (lane < r) sa.degen[k][lane] = dg[lane];
  if (lane == 0) sa.degen[k][r] = anyd;
}
__device__ void svd_fin2_warp(const SvdArgs& sa, int k) {
  __shared__ double scr[4 * RT_MAX_RANK * RT_MAX_RANK + 2 * RT_MAX_RANK];
  svd_fin2_warp_s(sa, k, scr, nullptr);
}

__global__ void __launch_bounds__(32) k_svd_fin2(SvdArgs sa) {
  if (rt_stopped(sa.stop)) return;
  if ((int)blockIdx.x < sa.n) svd_fin2_warp(sa, blockIdx.x);
}

// PH 3 tail: the fin2 step on H' = Q^T H Q (Q the Rayleigh-Ritz rotation, in
// r x r arithmetic instead of a second pass over the rotated Z), then T' = Q T so
// that the long side is Z T' straight from the unrotated projections.  `scr`:
// shared scratch of 6 r^2 + r doubles + 2 r ints.
__device__ void svd_fin2_ritz_warp(const SvdArgs& sa, int k, double* scr) {
  const int r = sa.r[k], lane = threadIdx.x & 31;
  double* q = scr;              // Q (r x r, column-major)
  double* hq = q + r * r;       // H Q
  double* hs = hq + r * r;      // H, then H'
  double* f2 = hs + r * r;      // fin2 scratch (4 r^2 + r doubles, 2 r ints)
  for (int e = lane; e < r * r; e += 32) {
    q[e] = sa.Q[k][e];
    hs[e] = sa.H[k][e];
  }
  __syncwarp();
  for (int e = lane; e < r * r; e += 32) {   // (H Q)[i, j]
    const int i = e % r, j = e / r;
    double v = 0.0;
    for (int p = 0; p < r; ++p) v = fma(hs[i + p * r], q[p + j * r], v);
    hq[e] = v;
  }
  __syncwarp();
  double hv[(RT_MAX_RANK * RT_MAX_RANK + 31) / 32];
  int nh = 0;
  for (int e = lane; e < r * r; e += 32, ++nh) {   // H' = Q^T (H Q), symmetrised
    const int i = e % r, j = e / r;
    const int a = min(i, j), b = max(i, j);
    double v = 0.0, w = 0.0;
    for (int p = 0; p < r; ++p) {
      v = fma(q[p + a * r], hq[p + b * r], v);
      w = fma(q[p + b * r], hq[p + a * r], w);
    }
    hv[nh] = 0.5 * (v + w);
  }
  __syncwarp();
  nh = 0;
  for (int e = lane; e < r * r; e += 32, ++nh) {
    hs[e] = hv[nh];
    sa.H[k][e] = hv[nh];
  }
  __syncwarp();
  svd_fin2_warp_s(sa, k, f2, hs);   // sa.Q <- T (also left at f2 + 2 r^2)
  const double* T = f2 + 2 * r * r;
  __syncwarp();
  for (int e = lane; e < r * r; e += 32) {   // T' = Q T, out
    const int i = e % r, j = e / r;
    double v = 0.0;
    for (int p = 0; p < r; ++p) v = fma(q[i + p * r], T[p + j * r], v);
    sa.Q[k][e] = v;
  }
}

// long-side vectors: out[t, a] = sum_b Z[t, b] T[b, a]; short side permuted in place later
__device__ void svd_complete_cta(const SvdArgs& sa, int k);
// the last CTA of each mode (ticket) then permutes the short side and completes
// degenerate columns (svd_complete_cta)
template <int R>
__global__ void __launch_bounds__(256) k_long(SvdArgs sa, unsigned int* counters) {
  if (rt_stopped(sa.stop)) return;
  __shared__ double ts[RT_MAX_RANK * RT_MAX_RANK];
  __shared__ bool am_last;
  const int k = blockIdx.y;
  if (k >= sa.n) return;
  const int r = sa.r[k];
  const i64 l = sa.l[k];
  const unsigned nch = (unsigned)((l + blockDim.x - 1) / blockDim.x);
  if ((i64)blockIdx.x * blockDim.x >= l) return;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) ts[i] = sa.Q[k][i];
  __syncthreads();
  const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < l) {
    const double* Z = sa.Z[k] + t * r;
    double z[R], o[R];
#pragma unroll
    for (int a = 0; a < R; ++a) { z[a] = a < r ? Z[a] : 0.0; o[a] = 0.0; }
#pragma unroll
    for (int b = 0; b < R; ++b)
#pragma unroll
      for (int a = 0; a < R; ++a)
        if (a < r && b < r) o[a] = fma(z[b], ts[b + a * r], o[a]);
    double* out = (sa.tall[k] ? sa.U[k] : sa.V[k]) + t * r;
#pragma unroll
    for (int a = 0; a < R; ++a)
      if (a < r) out[a] = o[a];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = (atomicAdd(&counters[k], 1u) == nch - 1);
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  if (threadIdx.x == 0) counters[k] = 0u;
  svd_complete_cta(sa, k);
}

// permute the short-side columns to the sigma order; complete degenerate
// columns of both sides with orthonormal vectors (only when sigma <= tau, where
// 1/sigma is dropped, so this never changes the low-rank iterate).
__device__ void svd_complete_cta(const SvdArgs& sa, int k) {
  __shared__ double tmp[RT_MAX_RANK];
  __shared__ double red[8];
  __shared__ double coef[RT_MAX_RANK];
  const int r = sa.r[k];
  const int s = sa.s[k];
  const i64 l = sa.l[k];
  double* S = sa.tall[k] ? sa.V[k] : sa.U[k];   // short side, s x r row-major
  double* Lg = sa.tall[k] ? sa.U[k] : sa.V[k];  // long side, l x r row-major
  // permute short side rows in place
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    double row[RT_MAX_RANK];
    for (int a = 0; a < r; ++a) row[a] = S[(i64)i * r + a];
    for (int a = 0; a < r; ++a) S[(i64)i * r + a] = row[sa.perm[k][a]];
  }
  __syncthreads();
  if (!sa.degen[k][r]) return;
  for (int side = 0; side < 2; ++side) {
    double* X = side == 0 ? Lg : S;
    const i64 len = side == 0 ? l : s;
    const bool short_side = side == 1;
    for (int a = 0; a < r; ++a) {
      // the short side from the eigensolver is orthonormal already
      if (short_side) break;
      if (!sa.degen[k][a]) continue;
      for (i64 c = 0; c < len; ++c) {
        // candidate e_c: residual norm^2 = 1 - sum_b X[c, b]^2 over valid columns b
        if (threadIdx.x == 0) {
          double nn = 1.0;
          for (int b = 0; b < r; ++b) {
            const bool valid = (b < a) || !sa.degen[k][b];
            coef[b] = (valid && b != a) ? X[c * r + b] : 0.0;
            nn -= coef[b] * coef[b];
          }
          tmp[0] = nn;
        }
        __syncthreads();
        const double nn = tmp[0];
        if (nn > 0.5) {
          const double inv = 1.0 / sqrt(nn);
          for (i64 t = threadIdx.x; t < len; t += blockDim.x) {
            double v = (t == c) ? 1.0 : 0.0;
            for (int b = 0; b < r; ++b) v -= coef[b] * X[t * r + b];
            X[t * r + a] = v * inv;
          }
          __syncthreads();
          break;
        }
        __syncthreads();
      }
    }
  }
  (void)red;
}

__global__ void __launch_bounds__(256) k_complete(SvdArgs sa) {
  if (rt_stopped(sa.stop)) return;
  if ((int)blockIdx.x < sa.n) svd_complete_cta(sa, blockIdx.x);
}
