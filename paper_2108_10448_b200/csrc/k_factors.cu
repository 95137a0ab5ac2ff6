// k_factors.cu -- the Tucker collapse of the fiber CUR:
//
//   reference (fiber_cur.py:264-267):  F_k = C_k @ pinv(U_k),  pinv = V S^+ U~^T
//   here:                              A_k = C_k V_k S_k^+      (d_k x r_k)
//                                      G   = core x_k U~_k^T     (r_1 x ... x r_n)
//   so core x_k F_k == G x_k A_k exactly (mode product with a product matrix).
//
// k_apass/k_areduce build A_k from the clean fibers (recomputed on the fly as
// x - HT(x - L_prev, zeta), bit-identical to the values the threshold pass
// produced); k_gpass/k_modeprod build G from the clean core; k_wcols builds
// the per-column weights W_b used by every block evaluation
//   L(p, q) = sum_a A_mode[row(p), a] W_b[q, a]
// (fiber_cur.py:288-326 evaluated in Tucker form, |J| r^n instead of |J| prod|I|).
#include "common.cuh"

struct APassArgs {
  const void* xb;
  int dtype;
  const double* st_s;               // state that produced the threshold (null: L = 0)
  double zeta;
  const double* V[RT_MAX_MODES];    // |J_k| x r row-major
  const double* siginv[RT_MAX_MODES];
  double* part;                     // [mode][chunks][d_max][r_max]
  int chunk;                        // columns per CTA
  int maxchunks;
  i64 dmax;
  double* st_out;                   // new state (A_k written at g.a_off[k])
};

template <int R>
__global__ void __launch_bounds__(256) k_apass(Geom g, IndexPtrs ip, APassArgs a) {
  __shared__ double vs[64 * RT_MAX_RANK];
  const int k = blockIdx.z;
  if (k >= g.n) return;
  const BlockDesc bd = g.blk[k + 1];
  const int r = bd.r;
  const i64 q0 = (i64)blockIdx.y * a.chunk;
  if (q0 >= bd.Q) return;
  const i64 q1 = min(bd.Q, q0 + a.chunk);
  const i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if ((i64)blockIdx.x * blockDim.x >= bd.P) return;
  double acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = 0.0;
  const double* V = a.V[k];
  for (i64 qs = q0; qs < q1; qs += 64) {
    const i64 qe = min(q1, qs + 64);
    __syncthreads();
    for (int i = threadIdx.x; i < (qe - qs) * r; i += blockDim.x) vs[i] = V[qs * r + i];
    __syncthreads();
    if (p < bd.P) {
      for (i64 q = qs; q < qe; ++q) {
        const double x = ld_elem(a.xb, bd.off + q * bd.P + p, a.dtype);
        const double ls = a.st_s ? eval_low(a.st_s, g, bd, ip.rows[0], p, q) : 0.0;
        const double c = x - hard_thr(x - ls, a.zeta);
        const double* vq = vs + (q - qs) * r;
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (i < r) acc[i] = fma(c, vq[i], acc[i]);
      }
    }
  }
  if (p < bd.P) {
    double* out = a.part + (((i64)k * a.maxchunks + blockIdx.y) * a.dmax + p) * RT_MAX_RANK;
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < r) out[i] = acc[i];
  }
}

// A_k[p, a] = siginv_a * sum over chunks (chunk order) of the partials
__global__ void k_areduce(Geom g, APassArgs a) {
  const int k = blockIdx.y;
  if (k >= g.n) return;
  const BlockDesc bd = g.blk[k + 1];
  const int r = bd.r;
  const int nch = (int)((bd.Q + a.chunk - 1) / a.chunk);
  double* A = a.st_out + g.a_off[k];
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < bd.P * r; e += (i64)gridDim.x * blockDim.x) {
    const i64 p = e % bd.P;
    const int i = (int)(e / bd.P);
    double acc = 0.0;
    const double* src = a.part + ((i64)k * a.maxchunks * a.dmax + p) * RT_MAX_RANK + i;
    for (int c = 0; c < nch; ++c) acc += src[(i64)c * a.dmax * RT_MAX_RANK];
    A[p + (i64)i * bd.P] = acc * a.siginv[k][i];
  }
}

// ------------------------------------------------------------------ G

struct GPassArgs {
  const void* xb;
  int dtype;
  const double* st_s;
  double zeta;
  const double* U[RT_MAX_MODES];   // |I_k| x r row-major
  double* t1;                       // r_1 x prod_{m>=2}|I_m| (F-order)
};

// first contraction of the clean core with U~_1^T (warp per core column)
template <int R>
__global__ void __launch_bounds__(256) k_gpass(Geom g, IndexPtrs ip, GPassArgs a) {
  const BlockDesc bd = g.blk[0];
  const int r = bd.r;
  const int lane = threadIdx.x & 31;
  const i64 q = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= bd.Q) return;
  double acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = 0.0;
  const double* U = a.U[0];
  for (i64 p = lane; p < bd.P; p += 32) {
    const double x = ld_elem(a.xb, bd.off + q * bd.P + p, a.dtype);
    const double ls = a.st_s ? eval_low(a.st_s, g, bd, ip.rows[0], p, q) : 0.0;
    const double c = x - hard_thr(x - ls, a.zeta);
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < r) acc[i] = fma(U[p * r + i], c, acc[i]);
  }
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = warp_sum(acc[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < r) a.t1[q * r + i] = acc[i];
  }
}

// out = in x_m U_m^T on the small partially-contracted core:
// in dims (r_1..r_{m-1}, |I_m|, |I_{m+1}|..), out dims (r_1..r_m, |I_{m+1}|..)
__global__ void k_modeprod(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ U,
                           i64 rho, int Im, int rm, i64 beta_n) {
  const i64 total = rho * rm * beta_n;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
    const i64 alpha = e % rho;
    const i64 rest = e / rho;
    const int aa = (int)(rest % rm);
    const i64 beta = rest / rm;
    double acc = 0.0;
    const double* src = in + alpha + rho * (i64)Im * beta;
    for (int i = 0; i < Im; ++i) acc = fma(U[(i64)i * rm + aa], src[rho * i], acc);
    out[e] = acc;
  }
}

// ------------------------------------------------------------------ W

// Per block column q: w[a] = sum over the other modes' rank indices of
//   G[a, beta] * prod_{m != mode} A_m[i_m(q), beta_m]
// full = 1: columns run over every (i_2..i_n) of the full tensor (K3 weights).
template <int R>
__global__ void __launch_bounds__(128) k_wcols(Geom g, IndexPtrs ip, double* __restrict__ st, int full,
                                              double* __restrict__ wfull) {
  extern __shared__ double gs[];
  const int b = blockIdx.y;
  BlockDesc bd;
  i64 Q;
  if (full) {
    bd = g.blk[0];
    Q = 1;
    for (int m = 1; m < g.n; ++m) Q *= g.dim[m];
  } else {
    if (b >= g.nblk) return;
    bd = g.blk[b];
    Q = bd.Q;
  }
  if ((i64)blockIdx.x * blockDim.x >= Q) return;
  for (i64 i = threadIdx.x; i < g.gsize; i += blockDim.x) gs[i] = st[i];
  __syncthreads();
  const i64 q = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  const int tgt = bd.mode;
  i64 idx[RT_MAX_MODES];
  if (full) {
    i64 t = q;
    for (int m = 1; m < g.n; ++m) { idx[m] = t % g.dim[m]; t /= g.dim[m]; }
  } else if (bd.is_core) {
    i64 t = q;
    for (int m = 1; m < g.n; ++m) {
      const i64 pos = t % g.nrows[m];
      t /= g.nrows[m];
      idx[m] = ip.rows[m][pos];
    }
  } else {
    i64 j = ip.cols[tgt][q];
    for (int m = 0; m < g.n; ++m) {
      if (m == tgt) continue;
      idx[m] = j % g.dim[m];
      j /= g.dim[m];
    }
  }
  const double* Abase[RT_MAX_MODES];
  for (int m = 0; m < g.n; ++m) Abase[m] = st + g.a_off[m] + (m == tgt ? 0 : idx[m]);
  double w[R];
#pragma unroll
  for (int i = 0; i < R; ++i) w[i] = 0.0;
  i64 combos = 1;
  for (int m = 0; m < g.n; ++m) if (m != tgt) combos *= g.rank[m];
  const int rt = g.rank[tgt];
  for (i64 c = 0; c < combos; ++c) {
    i64 t = c, goff = 0;
    double coef = 1.0;
    for (int m = 0; m < g.n; ++m) {
      if (m == tgt) continue;
      const int bm = (int)(t % g.rank[m]);
      t /= g.rank[m];
      goff += bm * g.gstride[m];
      coef *= Abase[m][(i64)bm * g.dim[m]];
    }
    const double* gp = gs + goff;
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < rt) w[i] = fma(gp[i * g.gstride[tgt]], coef, w[i]);
  }
  double* out = full ? wfull + q * rt : st + bd.w_off + q * rt;
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (i < rt) out[i] = w[i];
}

template __global__ void k_apass<4>(Geom, IndexPtrs, APassArgs);
template __global__ void k_apass<8>(Geom, IndexPtrs, APassArgs);
template __global__ void k_apass<16>(Geom, IndexPtrs, APassArgs);
template __global__ void k_apass<32>(Geom, IndexPtrs, APassArgs);
template __global__ void k_gpass<4>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<8>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<16>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<32>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_wcols<4>(Geom, IndexPtrs, double*, int, double*);
template __global__ void k_wcols<8>(Geom, IndexPtrs, double*, int, double*);
template __global__ void k_wcols<16>(Geom, IndexPtrs, double*, int, double*);
template __global__ void k_wcols<32>(Geom, IndexPtrs, double*, int, double*);
