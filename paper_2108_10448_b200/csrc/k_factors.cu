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
  int chunk;                        // columns per CTA (multiple of APASS_CH)
  int maxchunks;
  int pitch;                        // partial row pitch (the rank bucket)
  unsigned mode_mask;               // modes this launch handles (bit k)
  i64 dmax;
  double* st_out;                   // new state (A_k written at g.a_off[k])
};

#define APASS_CH 32   // fiber columns per CTA (V and W rows staged in shared memory)

template <int R>
__global__ void __launch_bounds__(256) k_apass(Geom g, IndexPtrs ip, APassArgs a) {
  __shared__ double vs[APASS_CH * R];
  __shared__ double wsh[APASS_CH * R];
  const int k = blockIdx.z;
  if (k >= g.n || !((a.mode_mask >> k) & 1u)) return;
  const BlockDesc& bd = g.blk[k + 1];
  const int r = bd.r;   // == R for the exact-rank launches (no dead unrolled terms)
  const i64 P = bd.P;
  const i64 q0 = (i64)blockIdx.y * a.chunk;
  if (q0 >= bd.Q) return;
  if ((i64)blockIdx.x * blockDim.x >= P) return;
  const int nq = (int)min((i64)a.chunk, bd.Q - q0);
  const double* V = a.V[k];
  const i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = p < P;
  // this row's A_prev entries are shared by every column of the chunk
  double arow[R];
#pragma unroll
  for (int i = 0; i < R; ++i) arow[i] = (live && a.st_s && i < r) ? a.st_s[g.a_off[k] + p + (i64)i * P] : 0.0;
  double acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = 0.0;
  for (int s0 = 0; s0 < nq; s0 += APASS_CH) {
    const int ns = min(APASS_CH, nq - s0);
    __syncthreads();
    for (int i = threadIdx.x; i < ns * r; i += blockDim.x) {
      vs[i] = V[(q0 + s0) * r + i];
      wsh[i] = a.st_s ? a.st_s[bd.w_off + (q0 + s0) * r + i] : 0.0;
    }
    __syncthreads();
    if (!live) continue;
    const i64 base = bd.off + (q0 + s0) * P + p;
    for (int q = 0; q < ns; q += 4) {
      double xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = (q + u < ns) ? ld_elem(a.xb, base + (i64)(q + u) * P, a.dtype) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (q + u >= ns) break;
        const double* wq = wsh + (q + u) * r;
        const double* vq = vs + (q + u) * r;
        double ls = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (i < r) ls = fma(arow[i], wq[i], ls);
        const double c = xv[u] - hard_thr(xv[u] - ls, a.zeta);
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (i < r) acc[i] = fma(c, vq[i], acc[i]);
      }
    }
  }
  if (!live) return;
  double* out = a.part + (((i64)k * a.maxchunks + blockIdx.y) * a.dmax + p) * a.pitch;
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (i < r) out[i] = acc[i];
}

// A_k[p, a] = siginv_a * sum over chunks (fixed warp-butterfly order) of the partials
__global__ void __launch_bounds__(256) k_areduce(Geom g, APassArgs a) {
  const int k = blockIdx.y;
  if (k >= g.n) return;
  const BlockDesc& bd = g.blk[k + 1];
  const int r = bd.r;
  const int nch = (int)((bd.Q + a.chunk - 1) / a.chunk);
  double* A = a.st_out + g.a_off[k];
  const int lane = threadIdx.x & 31;
  const i64 nout = bd.P * r;
  for (i64 o = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < nout; o += ((i64)gridDim.x * blockDim.x) >> 5) {
    const i64 p = o % bd.P;
    const int i = (int)(o / bd.P);
    const double* src = a.part + ((i64)k * a.maxchunks * a.dmax + p) * a.pitch + i;
    double acc = 0.0;
    for (int c = lane; c < nch; c += 32) acc += src[(i64)c * a.dmax * a.pitch];
    acc = warp_sum(acc);
    if (lane == 0) A[p + (i64)i * bd.P] = acc * a.siginv[k][i];
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
__global__ void __launch_bounds__(256) k_modeprod(const double* __restrict__ in, double* __restrict__ out,
                                                   const double* __restrict__ U, i64 rho, int Im, int rm, i64 beta_n) {
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
                                                       i64 d, i64 rho, i64 Pm, int rm, i64 beta_n) {
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

// ------------------------------------------------------------------ W

// Per block column q: w[a] = sum over the other modes' rank indices of
//   G[a, beta] * prod_{m != mode} A_m[i_m(q), beta_m]
// full = 1: columns run over every (i_2..i_n) of the full tensor (K3 weights).
// dynamic shared memory: G (gsize doubles) + per thread the other modes' A rows
template <int R>
__global__ void __launch_bounds__(128) k_wcols(Geom g, IndexPtrs ip, double* __restrict__ st, int full,
                                              double* __restrict__ wfull, int rows_per_thread, int skip_core) {
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

template __global__ void k_apass<4>(Geom, IndexPtrs, APassArgs);
template __global__ void k_apass<8>(Geom, IndexPtrs, APassArgs);
template __global__ void k_apass<16>(Geom, IndexPtrs, APassArgs);
template __global__ void k_apass<32>(Geom, IndexPtrs, APassArgs);
template __global__ void k_gpass<4>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<8>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<16>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_gpass<32>(Geom, IndexPtrs, GPassArgs);
template __global__ void k_wcols<4>(Geom, IndexPtrs, double*, int, double*, int, int);
template __global__ void k_wcols<8>(Geom, IndexPtrs, double*, int, double*, int, int);
template __global__ void k_wcols<16>(Geom, IndexPtrs, double*, int, double*, int, int);
template __global__ void k_wcols<32>(Geom, IndexPtrs, double*, int, double*, int, int);
