// k_factors.cu -- the Tucker collapse of the fiber CUR:
//
//   reference (fiber_cur.py:264-267):  F_k = C_k @ pinv(U_k),  pinv = V S^+ U~^T
//   here:                              A_k = C_k V_k S_k^+      (d_k x r_k)
//                                      G   = core x_k U~_k^T     (r_1 x ... x r_n)
//   so core x_k F_k == G x_k A_k exactly (mode product with a product matrix).
//
// The A pass (k_block_pass<..AP>, bp_pass.cuh) builds A_k from the clean fibers (recomputed on the fly as
// x - HT(x - L_prev, zeta), bit-identical to the values the threshold pass
// produced); k_gpass/k_modeprod build G from the clean core; k_wcols builds
// the per-column weights W_b used by every block evaluation
//   L(p, q) = sum_a A_mode[row(p), a] W_b[q, a]
// (fiber_cur.py:288-326 evaluated in Tucker form, |J| r^n instead of |J| prod|I|).
#include "common.cuh"


// ------------------------------------------------------------------ G

struct GPassArgs {
  const void* xb;
  int dtype;
  const double* st_s;
  double zeta;
  const double* zetap;             // if set: zeta from device memory
  const double* U[RT_MAX_MODES];   // |I_k| x r row-major
  double* t1;                       // r_1 x prod_{m>=2}|I_m| (F-order)
};

// first contraction of the clean core with U~_1^T (warp per core column)
template <int R>
__global__ void __launch_bounds__(256) k_gpass(Geom g, IndexPtrs ip, GPassArgs a) {
  if (rt_stopped(g.stop)) return;
  const BlockDesc bd = g.blk[0];
  const int r = bd.r;
  const int lane = threadIdx.x & 31;
  const i64 q = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= bd.Q) return;
  double acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = 0.0;
  const double* U = a.U[0];
  const double zeta = a.zetap ? __ldg(a.zetap) : a.zeta;
  for (i64 p = lane; p < bd.P; p += 32) {
    const double x = ld_elem(a.xb, bd.off + q * bd.P + p, a.dtype);
    const double ls = a.st_s ? eval_low(a.st_s, g, bd, ip.rows[0], p, q) : 0.0;
    const double c = x - hard_thr(x - ls, zeta);
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
__global__ void __launch_bounds__(256) k_modeprod(const double* __restrict__ in, double* __restrict__ out,
                                                   const double* __restrict__ U, i64 rho, int Im, int rm, i64 beta_n,
                                                   const int* __restrict__ stop) {
  if (rt_stopped(stop)) return;
  const i64 total = rho * rm * beta_n;
  const int lane = threadIdx.x & 31;
  for (i64 e = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < total; e += ((i64)gridDim.x * blockDim.x) >> 5) {
    const i64 alpha = e % rho;
    const i64 rest = e / rho;
    const int aa = (int)(rest % rm);
    const i64 beta = rest / rm;
    const double* src = in + alpha + rho * (i64)Im * beta;
    double acc = 0.0;
    for (int i = lane; i < Im; i += 32) acc = fma(U[(i64)i * rm + aa], src[rho * i], acc);
    acc = warp_sum(acc);
    if (lane == 0) out[e] = acc;
  }
}

// out = in x_m B with B[p, b] = A[row(p) + b * d] (row(p) = rows[p] or p):
// in dims (rho, r_m, beta_n), out dims (rho, Pm, beta_n) -- the expanding mode
// product used to build W_core = G x_{m>=2} A_m(I_m, :) and the full-tensor
// weights Tf = G x_{m>=2} A_m as a chain (cost r_m per output instead of
// prod r per column).
__global__ void __launch_bounds__(256) k_modeprod_fwd(const double* __restrict__ in, double* __restrict__ out,
                                                       const double* __restrict__ A, const int* __restrict__ rows,
                                                       i64 d, i64 rho, i64 Pm, int rm, i64 beta_n,
                                                       const int* __restrict__ stop) {
  if (rt_stopped(stop)) return;
  const i64 total = rho * Pm * beta_n;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
    const i64 alpha = e % rho;
    const i64 rest = e / rho;
    const i64 p = rest % Pm;
    const i64 beta = rest / Pm;
    const double* src = in + alpha + rho * (i64)rm * beta;
    const double* arow = A + (rows ? (i64)rows[p] : p);
    double acc = 0.0;
    for (int b = 0; b < rm; ++b) acc = fma(arow[(i64)b * d], src[rho * b], acc);
    out[e] = acc;
  }
}

// Warp per block column: w[a] = sum over the other modes' rank combinations c of
//   G[a, c] * prod_{m != t} A_m[i_m(q), c_m]
// with the combinations split over the lanes (a per-block table of G offsets and
// per-mode indices, built once per CTA in shared memory), the other modes' A rows
// of the column staged per warp, and a fixed-order butterfly sum of the r_t
// partials.  Dynamic shared memory: G | goff[ncombo] (int) | cidx[ncombo][n-1]
// (uchar) | per warp 32 * ceil(sum r_other / 32) row values.
// GS lanes per column (32: one warp; 8: four columns per warp for geometries with
// few combinations, e.g. 25 at n = 3, r = 5).
#define WC_WARPS 8
template <int R, int GS>
__global__ void __launch_bounds__(32 * WC_WARPS) k_wcols_warp(Geom g, IndexPtrs ip, double* __restrict__ st,
                                                             int skip_core, int rows_cap) {
  if (rt_stopped(g.stop)) return;
  constexpr int NG = 32 * WC_WARPS / GS;   // column groups per CTA
  extern __shared__ double wsm[];
  const int b = blockIdx.y;
  if (b >= g.nblk || (skip_core && g.blk[b].is_core)) return;
  const BlockDesc& bd = g.blk[b];
  const i64 Q = bd.Q;
  if ((i64)blockIdx.x * NG >= Q) return;
  const int tgt = bd.mode, rt = g.rank[tgt];
  const i64 gst = g.gstride[tgt];
  int no = 0, ncombo = 1, rsum = 0;
  int om[RT_MAX_MODES], ro[RT_MAX_MODES];
  for (int m = 0; m < g.n; ++m) {
    if (m == tgt) continue;
    om[no] = m;
    ro[no] = rsum;
    rsum += g.rank[m];
    ncombo *= g.rank[m];
    ++no;
  }
  double* G = wsm;
  int* goff = reinterpret_cast<int*>(G + g.gsize);
  unsigned char* cidx = reinterpret_cast<unsigned char*>(goff + ncombo);
  double* rows = G + g.gsize + ((size_t)ncombo * 4 + (size_t)ncombo * (no > 0 ? no : 1) + 7) / 8 + 1;
  for (i64 i = threadIdx.x; i < g.gsize; i += blockDim.x) G[i] = st[i];
  for (int c = threadIdx.x; c < ncombo; c += blockDim.x) {
    int t = c, off = 0;
    for (int j = 0; j < no; ++j) {   // first other mode fastest
      const int rk = g.rank[om[j]];
      const int ij = t % rk;
      t /= rk;
      off += ij * (int)g.gstride[om[j]];
      cidx[(size_t)c * no + j] = (unsigned char)ij;
    }
    goff[c] = off;
  }
  __syncthreads();
  const int lane = threadIdx.x % GS, w = threadIdx.x / GS;
  const unsigned gmask = GS == 32 ? 0xffffffffu : (((1u << GS) - 1u) << ((threadIdx.x & 31) & ~(GS - 1)));
  double* rb = rows + (size_t)w * rows_cap;
  for (i64 q = (i64)blockIdx.x * NG + w; q < Q; q += (i64)gridDim.x * NG) {
    // the other modes' A rows of this column
    {
      i64 t = q, j = bd.is_core ? 0 : ip.cols[tgt][q];
      for (int k = 0; k < no; ++k) {
        const int m = om[k];
        i64 im;
        if (bd.is_core) {
          const i64 pos = t % g.nrows[m];
          t /= g.nrows[m];
          im = ip.rows[m][pos];
        } else {
          // fiber columns enumerate the other modes ascending, first fastest (tensor.py:250-283)
          im = j % g.dim[m];
          j /= g.dim[m];
        }
        for (int bm = lane; bm < g.rank[m]; bm += GS) rb[ro[k] + bm] = st[g.a_off[m] + im + (i64)bm * g.dim[m]];
      }
    }
    __syncwarp(gmask);
    double acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = 0.0;
    for (int c = lane; c < ncombo; c += GS) {
      double coef = 1.0;
      for (int k = no - 1; k >= 0; --k) coef *= rb[ro[k] + cidx[(size_t)c * no + k]];
      const double* gq = G + goff[c];
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i < rt) acc[i] = fma(gq[i * gst], coef, acc[i]);
    }
    double* out = st + bd.w_off + q * rt;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (i < rt) {
        double v = acc[i];
#pragma unroll
        for (int o = GS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);   // fixed order
        if (lane == 0) out[i] = v;
      }
    }
    __syncwarp(gmask);
  }
}

// ------------------------------------------------------------------ W

// Per block column q: w[a] = sum over the other modes' rank indices of
//   G[a, beta] * prod_{m != mode} A_m[i_m(q), beta_m]
// full = 1: columns run over every (i_2..i_n) of the full tensor (K3 weights).
// dynamic shared memory: G (gsize doubles) + per thread the other modes' A rows
template <int R>
__global__ void __launch_bounds__(128) k_wcols(Geom g, IndexPtrs ip, double* __restrict__ st, int full,
                                              double* __restrict__ wfull, int rows_per_thread, int skip_core) {
  if (rt_stopped(g.stop)) return;
  extern __shared__ double gsm[];
  const int b = blockIdx.y;
  i64 Q;
  int tgt, is_core;
  i64 w_off;
  if (full) {
    Q = 1;
    for (int m = 1; m < g.n; ++m) Q *= g.dim[m];
    tgt = 0;
    is_core = 1;
    w_off = 0;
  } else {
    if (b >= g.nblk || (skip_core && g.blk[b].is_core)) return;
    Q = g.blk[b].Q;
    tgt = g.blk[b].mode;
    is_core = g.blk[b].is_core;
    w_off = g.blk[b].w_off;
  }
  if ((i64)blockIdx.x * blockDim.x >= Q) return;
  for (i64 i = threadIdx.x; i < g.gsize; i += blockDim.x) gsm[i] = st[i];
  double* rowbuf = gsm + g.gsize + (i64)threadIdx.x * rows_per_thread;
  __syncthreads();
  const i64 q = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  // gather the A_m rows of the other modes (independent loads, all in flight)
  {
    i64 t = q, j = 0;
    if (!full && !is_core) j = ip.cols[tgt][q];
    int o = 0;
    for (int m = 0; m < g.n; ++m) {
      if (m == tgt) continue;
      i64 im;
      if (full) {
        im = t % g.dim[m];
        t /= g.dim[m];
      } else if (is_core) {
        const i64 pos = t % g.nrows[m];
        t /= g.nrows[m];
        im = ip.rows[m][pos];
      } else {
        im = j % g.dim[m];
        j /= g.dim[m];
      }
      const double* Am = st + g.a_off[m] + im;
      for (int bm = 0; bm < g.rank[m]; ++bm) rowbuf[o + bm] = Am[(i64)bm * g.dim[m]];
      o += g.rank[m];
    }
  }
  double w[R];
#pragma unroll
  for (int i = 0; i < R; ++i) w[i] = 0.0;
  // odometer over the other modes' rank indices (first other mode fastest):
  // suffix products pp[j] = prod_{l >= j} rows_l[idx_l] and the G offset are
  // updated incrementally, so a combination costs r_t FMAs + O(1)
  int om[RT_MAX_MODES], rk[RT_MAX_MODES], ro[RT_MAX_MODES], ix[RT_MAX_MODES];
  i64 gs[RT_MAX_MODES];
  int no = 0;
  {
    int o = 0;
    for (int m = 0; m < g.n; ++m) {
      if (m == tgt) continue;
      om[no] = m;
      rk[no] = g.rank[m];
      ro[no] = o;
      gs[no] = g.gstride[m];
      ix[no] = 0;
      o += g.rank[m];
      ++no;
    }
  }
  double pp[RT_MAX_MODES + 1];
  pp[no] = 1.0;
  for (int j = no - 1; j >= 0; --j) pp[j] = pp[j + 1] * rowbuf[ro[j]];
  i64 goff = 0;
  const int rt = g.rank[tgt];
  const i64 gst = g.gstride[tgt];
  while (true) {
    const double coef = pp[0];
    const double* gq = gsm + goff;
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < rt) w[i] = fma(gq[i * gst], coef, w[i]);
    // increment the odometer
    int j = 0;
    while (j < no) {
      ++ix[j];
      goff += gs[j];
      if (ix[j] < rk[j]) break;
      goff -= gs[j] * rk[j];
      ix[j] = 0;
      ++j;
    }
    if (j == no) break;
    // refresh the suffix products of positions <= j
    for (int l = j; l >= 0; --l) pp[l] = pp[l + 1] * rowbuf[ro[l] + ix[l]];
  }
  (void)om;
  double* out = full ? wfull + q * rt : st + w_off + q * rt;
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (i < rt) out[i] = w[i];
}

template __global__ void k_gpass<4>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<8>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<16>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<32>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_wcols<4>(Geom, IndexPtrs, double*, int, double*, int, int);
template __global__ void k_wcols_warp<4, 32>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols_warp<8, 32>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols_warp<16, 32>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols_warp<32, 32>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols_warp<4, 8>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols_warp<8, 8>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols_warp<16, 8>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols_warp<32, 8>(Geom, IndexPtrs, double*, int, int);
template __global__ void k_wcols<8>(Geom, IndexPtrs, double*, int, double*, int, int);
template __global__ void k_wcols<16>(Geom, IndexPtrs, double*, int, double*, int, int);
template __global__ void k_wcols<32>(Geom, IndexPtrs, double*, int, double*, int, int);
