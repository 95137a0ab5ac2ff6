// bp_pass.cuh -- the persistent K1 block pass (template definition).  Explicitly
// instantiated per rank bucket in bp_rb{4,8,16,32}.cu so the variants compile in
// parallel; engine.cu/k_block.cu see only the declaration in k_block.cu.
#pragma once
#include "bp_types.cuh"

// Per-tile operands of the block pass.  A tile is `ncols` whole columns of one
// block (P rows each) staged in shared memory: x (column-major, tile-local)
// and the columns' W rows of both states (row-major, r per column).  A rows
// are read through L1 from the state (column-major, stride d; core rows via I_1).
struct BPTile {
  const unsigned char* x;  // staged x (dtype), already offset by the 16-byte skip
  int dtype;
  int P, ncols, r;
  const double* As;        // A_mode of the threshold state (global) or null
  const double* Ae;        // A_mode of the error state (global) or null
  i64 d;                   // A column stride
  const int* rows0;        // core: I_1 (0-based); fibers: null
  const double* Wss;       // smem W rows, threshold state
  const double* Wes;       // smem W rows, error state
  const int* rmap;         // smem rowpos of the fiber mode (-1: row not in I_k)
  const double* Asm;       // lanes over columns: the block's A rows (threshold state), smem, row pitch apitch
  const double* Aem;       // same for the error state
  int apitch;
  double* Mk;              // intersection output at the tile's first column (column-major, mrows)
  int mrows;
  double zeta;
  double *s_out, *c_out, *l_out;   // exports at the tile's first element
  const double* U;         // G pass: U~_1 (|I_1| x r row-major)
  double* t1;              // G pass: output rows at the tile's first column
  double* gp;              // G pass: smem partials
};

__device__ __forceinline__ double bp_x(const BPTile& T, int i) {
  return T.dtype == 0 ? reinterpret_cast<const double*>(T.x)[i] : (double)reinterpret_cast<const float*>(T.x)[i];
}

// One entry: threshold against state s, clean value, intersection scatter, error
// against state e, exports, and the sums.  Returns the clean value.
template <bool HS, bool HE, bool WM, bool EXP>
__device__ __forceinline__ double bp_entry(const BPTile& T, double x, double ls, double le, int pos, int ql, int p,
                                           double& e2, double& x2, bool& bad) {
  const double sv = fabs(x - ls) <= T.zeta ? 0.0 : x - ls;
  const double c = x - sv;
  if (WM && pos >= 0) {
    T.Mk[pos + (i64)ql * T.mrows] = c;
    bad |= !isfinite(c);
  }
  if (HE) {
    const double rr = x - le - sv;
    e2 = fma(rr, rr, e2);
  }
  if (EXP) {
    const int k = ql * T.P + p;
    if (T.s_out) T.s_out[k] = sv;
    if (T.c_out) T.c_out[k] = c;
    if (T.l_out) T.l_out[k] = le;
  }
  x2 = fma(x, x, x2);
  return c;
}

template <int DT>
__device__ __forceinline__ double bp_xt(const unsigned char* x, int i) {
  return DT == 0 ? reinterpret_cast<const double*>(x)[i] : (double)reinterpret_cast<const float*>(x)[i];
}

// A row dot W row with R terms; A row from shared memory (even pitch, 16-byte aligned)
template <int R, bool EX>
__device__ __forceinline__ double bp_dot_sm(const double* __restrict__ arow, const double* w, int r) {
  double acc = 0.0;
#pragma unroll
  for (int kk = 0; kk < R; kk += 2) {
    const double2 a2 = *reinterpret_cast<const double2*>(arow + kk);
    if (EX || kk < r) acc = fma(a2.x, w[kk], acc);
    if (kk + 1 < R && (EX || kk + 1 < r)) acc = fma(a2.y, w[kk + 1], acc);
  }
  return acc;
}

// Lanes over columns (tiles of 32 * 2^k columns, small P): each lane keeps its
// column's W rows in registers; the warps split the tile into (32-column group,
// row range) items (the planner makes the group count divide the 8 warps) and
// the block's A rows come from shared memory as warp-broadcast loads.
// GP: the G pass -- t1[q, :] = sum_p U~_1[p, :] clean(p, q) on the core,
// with the row-range partials combined in fixed order through shared memory.
template <int R, bool EX, int DT, bool HS, bool HE, bool WM, bool EXP, bool GP>
__device__ __forceinline__ void bp_cols(const BPTile& T, double& e2, double& x2, bool& bad) {
  const int r = EX ? R : T.r;   // EX: the block rank is exactly R, else r <= R
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int P = T.P, ncols = T.ncols, ap = T.apitch;
  const int ncg = (ncols + 31) >> 5;
  const int nrr = max(1, nw / ncg);
  const int rlen = (P + nrr - 1) / nrr;
  const int items = ncg * nrr;
#pragma unroll 1
  for (int it = w; it < items; it += nw) {
    const int cg = it % ncg, rr = it / ncg;
    const int ql = cg * 32 + lane;
    const bool valid = ql < ncols;
    double ws[R], we[R], acc[R];
#pragma unroll
    for (int kk = 0; kk < R; ++kk) {
      const bool on = valid && (EX || kk < r);
      ws[kk] = (HS && on) ? T.Wss[ql * r + kk] : 0.0;
      we[kk] = (HE && on) ? T.Wes[ql * r + kk] : 0.0;
      acc[kk] = 0.0;
    }
    const int pb = rr * rlen, pe = min(P, pb + rlen);
    const int qoff = (valid ? ql : 0) * P;
    // one row's entry: threshold/error/exports, then the G-pass accumulation
    auto row_step = [&](int p, double x, double ls, double le) {
      const int pos = WM ? T.rmap[p] : -1;
      double c = 0.0;
      if (valid) c = bp_entry<HS, HE, WM, EXP>(T, x, ls, le, pos, ql, p, e2, x2, bad);
      if (GP) {
        const double* u = T.Aem + p * ap;   // U~_1 row p (staged, even pitch)
#pragma unroll
        for (int kk = 0; kk < R; kk += 2) {
          const double2 u2 = *reinterpret_cast<const double2*>(u + kk);
          if (EX || kk < r) acc[kk] = fma(u2.x, c, acc[kk]);
          if (kk + 1 < R && (EX || kk + 1 < r)) acc[kk + 1] = fma(u2.y, c, acc[kk + 1]);
        }
      }
    };
    // two rows per step: their dot products are independent chains; the entries
    // are then applied in row order, so every sum is bit-identical to the row loop
    int p = pb;
#pragma unroll 1
    for (; p + 1 < pe; p += 2) {
      const double x0 = bp_xt<DT>(T.x, qoff + p), x1 = bp_xt<DT>(T.x, qoff + p + 1);
      const double ls0 = HS ? bp_dot_sm<R, EX>(T.Asm + p * ap, ws, r) : 0.0;
      const double ls1 = HS ? bp_dot_sm<R, EX>(T.Asm + (p + 1) * ap, ws, r) : 0.0;
      const double le0 = HE ? bp_dot_sm<R, EX>(T.Aem + p * ap, we, r) : 0.0;
      const double le1 = HE ? bp_dot_sm<R, EX>(T.Aem + (p + 1) * ap, we, r) : 0.0;
      row_step(p, x0, ls0, le0);
      row_step(p + 1, x1, ls1, le1);
    }
    if (p < pe) {
      const double x = bp_xt<DT>(T.x, qoff + p);
      const double ls = HS ? bp_dot_sm<R, EX>(T.Asm + p * ap, ws, r) : 0.0;
      const double le = HE ? bp_dot_sm<R, EX>(T.Aem + p * ap, we, r) : 0.0;
      row_step(p, x, ls, le);
    }
    if (GP) {
      if (nrr == 1) {
        if (valid)
#pragma unroll
          for (int kk = 0; kk < R; ++kk)
            if (EX || kk < r) T.t1[(i64)ql * r + kk] = acc[kk];
      } else {
#pragma unroll
        for (int kk = 0; kk < R; ++kk)
          if (EX || kk < r) T.gp[((i64)rr * ncg * 32 + ql) * r + kk] = acc[kk];
      }
    }
  }
  if (GP && nrr > 1) {
    __syncthreads();
    for (int o = threadIdx.x; o < ncols * r; o += blockDim.x) {
      double s = 0.0;
      for (int rr = 0; rr < nrr; ++rr) s += T.gp[(i64)rr * ncg * 32 * r + o];   // fixed order
      T.t1[o] = s;
    }
  }
}

// Lanes over rows (tall tiles): items are (32-row chunk, column) pairs in
// chunk-major order and each warp takes a contiguous run of them, so a lane
// keeps the A rows of its row p in registers across the run (reloaded only at
// a chunk change) and each column's W row is a warp-broadcast shared load.
template <int R, bool EX, int DT, bool HS, bool HE, bool WM, bool EXP>
__device__ __forceinline__ void bp_rows(const BPTile& T, double& e2, double& x2, bool& bad) {
  const int r = EX ? R : T.r;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int P = T.P, ncols = T.ncols;
  const int nrc = (P + 31) >> 5;
  const int items = nrc * ncols;
  const int i0 = items * w / nw, i1 = items * (w + 1) / nw;
  // the warp's run [i0, i1) as segments of one row chunk each
#pragma unroll 1
  for (int it = i0; it < i1;) {
    const int rc = it / ncols, qb = it - rc * ncols;
    const int qe = min(ncols, qb + (i1 - it));
    it += qe - qb;
    const int p = rc * 32 + lane;
    if (p >= P) continue;
    const i64 grow = T.rows0 ? (i64)T.rows0[p] : (i64)p;
    double as[R], ae[R];
#pragma unroll
    for (int kk = 0; kk < R; ++kk) {
      const bool on = EX || kk < r;
      as[kk] = (HS && on) ? __ldg(T.As + grow + (i64)kk * T.d) : 0.0;
      ae[kk] = (HE && on) ? __ldg(T.Ae + grow + (i64)kk * T.d) : 0.0;
    }
    const int pos = WM ? T.rmap[p] : -1;
    // two columns per step: independent FMA chains (each in kk order, so every
    // entry's value is bit-identical to the one-column loop)
    int q = qb;
#pragma unroll 1
    for (; q + 1 < qe; q += 2) {
      const double x0 = bp_xt<DT>(T.x, q * P + p), x1 = bp_xt<DT>(T.x, (q + 1) * P + p);
      const double* ws0 = T.Wss + q * r;
      const double* we0 = T.Wes + q * r;
      double ls0 = 0.0, le0 = 0.0, ls1 = 0.0, le1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < R; ++kk) {
        if (EX || kk < r) {
          if (HS) {
            ls0 = fma(as[kk], ws0[kk], ls0);
            ls1 = fma(as[kk], ws0[r + kk], ls1);
          }
          if (HE) {
            le0 = fma(ae[kk], we0[kk], le0);
            le1 = fma(ae[kk], we0[r + kk], le1);
          }
        }
      }
      bp_entry<HS, HE, WM, EXP>(T, x0, ls0, le0, pos, q, p, e2, x2, bad);
      bp_entry<HS, HE, WM, EXP>(T, x1, ls1, le1, pos, q + 1, p, e2, x2, bad);
    }
    if (q < qe) {
      const double x = bp_xt<DT>(T.x, q * P + p);
      const double* wsr = T.Wss + q * r;
      const double* wer = T.Wes + q * r;
      double ls = 0.0, le = 0.0;
#pragma unroll
      for (int kk = 0; kk < R; ++kk) {
        if (EX || kk < r) {
          if (HS) ls = fma(as[kk], wsr[kk], ls);
          if (HE) le = fma(ae[kk], wer[kk], le);
        }
      }
      bp_entry<HS, HE, WM, EXP>(T, x, ls, le, pos, q, p, e2, x2, bad);
    }
  }
}

// A pass: A_new[p, :] += sum_q clean(p, q) V[q, :] over the tile's columns.
// Warp w owns the 32-row chunks rc = w (mod warps), the same rows in every tile,
// so the per-block shared accumulator acc[p * r + a] has a single writer per row.
template <int R, bool EX, int DT, bool HS>
__device__ __forceinline__ void bp_apass(const BPTile& T, double* __restrict__ acc) {
  const int r = EX ? R : T.r;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int P = T.P, ncols = T.ncols;
  const int nrc = (P + 31) >> 5;
#pragma unroll 1
  for (int rc = w; rc < nrc; rc += nw) {
    const int p = rc * 32 + lane;
    if (p >= P) continue;
    double as[R], ar[R];
#pragma unroll
    for (int kk = 0; kk < R; ++kk) {
      as[kk] = (HS && (EX || kk < r)) ? __ldg(T.As + p + (i64)kk * T.d) : 0.0;
      ar[kk] = 0.0;
    }
    // two columns per step: independent threshold chains (each in the threshold
    // pass's kk order, so the clean values are bit-identical to it)
    int q = 0;
#pragma unroll 1
    for (; q + 1 < ncols; q += 2) {
      const double x0 = bp_xt<DT>(T.x, q * P + p), x1 = bp_xt<DT>(T.x, (q + 1) * P + p);
      const double* w0 = T.Wss + q * r;
      const double* v0 = T.Wes + q * r;   // V rows are staged in the second W slot
      double l0 = 0.0, l1 = 0.0;
      if (HS) {
#pragma unroll
        for (int kk = 0; kk < R; ++kk)
          if (EX || kk < r) {
            l0 = fma(as[kk], w0[kk], l0);
            l1 = fma(as[kk], w0[r + kk], l1);
          }
      }
      const double c0 = x0 - hard_thr(x0 - l0, T.zeta), c1 = x1 - hard_thr(x1 - l1, T.zeta);
#pragma unroll
      for (int kk = 0; kk < R; ++kk)
        if (EX || kk < r) ar[kk] = fma(c1, v0[r + kk], fma(c0, v0[kk], ar[kk]));
    }
    if (q < ncols) {
      const double x = bp_xt<DT>(T.x, q * P + p);
      const double* wsr = T.Wss + q * r;
      const double* vr = T.Wes + q * r;
      double ls = 0.0;
      if (HS) {
#pragma unroll
        for (int kk = 0; kk < R; ++kk)
          if (EX || kk < r) ls = fma(as[kk], wsr[kk], ls);
      }
      const double c = x - hard_thr(x - ls, T.zeta);
#pragma unroll
      for (int kk = 0; kk < R; ++kk)
        if (EX || kk < r) ar[kk] = fma(c, vr[kk], ar[kk]);
    }
    double* ap = acc + (i64)p * r;
#pragma unroll
    for (int kk = 0; kk < R; ++kk)
      if (EX || kk < r) ap[kk] += ar[kk];
  }
}

template <int RR, int RB, bool HS>
__device__ __forceinline__ bool bp_try_ap(const BPTile& T, double* acc) {
  if (RR > RB || 2 * RR <= RB || T.r != RR) return false;
  constexpr int R = RR <= RB ? RR : RB;
  if (T.dtype == 0) bp_apass<R, true, 0, HS>(T, acc);
  else bp_apass<R, true, 1, HS>(T, acc);
  return true;
}

template <int RB, bool HS>
__device__ __forceinline__ void bp_tile_ap(const BPTile& T, double* acc) {
  if (bp_try_ap<1, RB, HS>(T, acc)) return;
  if (bp_try_ap<2, RB, HS>(T, acc)) return;
  if (bp_try_ap<3, RB, HS>(T, acc)) return;
  if (bp_try_ap<4, RB, HS>(T, acc)) return;
  if (bp_try_ap<5, RB, HS>(T, acc)) return;
  if (bp_try_ap<6, RB, HS>(T, acc)) return;
  if (bp_try_ap<8, RB, HS>(T, acc)) return;
  if (bp_try_ap<10, RB, HS>(T, acc)) return;
  if (bp_try_ap<16, RB, HS>(T, acc)) return;
  if (T.dtype == 0) bp_apass<RB, false, 0, HS>(T, acc);
  else bp_apass<RB, false, 1, HS>(T, acc);
}

template <int RR, int RB, bool HS, bool HE, bool WM, bool EXP, bool GP>
__device__ __forceinline__ bool bp_try(const BPTile& T, bool cols, double& e2, double& x2, bool& bad) {
  if (RR > RB || 2 * RR <= RB || T.r != RR) return false;   // exact ranks in (RB/2, RB]
  constexpr int R = RR <= RB ? RR : RB;
  if (cols) {
    if (T.dtype == 0) bp_cols<R, true, 0, HS, HE, WM, EXP, GP>(T, e2, x2, bad);
    else bp_cols<R, true, 1, HS, HE, WM, EXP, GP>(T, e2, x2, bad);
  } else if (!GP) {
    if (T.dtype == 0) bp_rows<R, true, 0, HS, HE, WM, EXP>(T, e2, x2, bad);
    else bp_rows<R, true, 1, HS, HE, WM, EXP>(T, e2, x2, bad);
  }
  return true;
}

// exact-rank specialisations in the kernel's rank bucket (RB/2, RB], else r <= RB at run time
template <int RB, bool HS, bool HE, bool WM, bool EXP, bool GP>
__device__ __forceinline__ void bp_tile_r(const BPTile& T, bool cols, double& e2, double& x2, bool& bad) {
  if (bp_try<1, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<2, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<3, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<4, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<5, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<6, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<8, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<10, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (bp_try<16, RB, HS, HE, WM, EXP, GP>(T, cols, e2, x2, bad)) return;
  if (cols) {
    if (T.dtype == 0) bp_cols<RB, false, 0, HS, HE, WM, EXP, GP>(T, e2, x2, bad);
    else bp_cols<RB, false, 1, HS, HE, WM, EXP, GP>(T, e2, x2, bad);
  } else if (!GP) {
    if (T.dtype == 0) bp_rows<RB, false, 0, HS, HE, WM, EXP>(T, e2, x2, bad);
    else bp_rows<RB, false, 1, HS, HE, WM, EXP>(T, e2, x2, bad);
  }
}

// Persistent K1 block pass.  CTA c processes a contiguous range of tiles of
// the compact blocks (tiles are whole columns of one block, so x and the
// columns' W rows are contiguous).  Each tile's x, W_s, W_e ranges are
// streamed into a shared-memory ring by cp.async.bulk (one mbarrier per
// stage).  Per entry -- L = A[row] . W[col] (r FMAs per state), hard
// threshold, clean value, intersection scatter, error sums -- with the lane
// mapping chosen per block (TileMap::cols): lanes over columns for short
// blocks, lanes over rows for tall ones.  Per-(CTA, block) partial sums are
// combined by the last CTA in CTA order (deterministic: the tile -> CTA
// assignment is static).  GP: the G pass over the core block's tiles only.
template <bool HS, bool HE, bool WM, bool EXP, bool GP, int RB, bool AP>
__global__ void __launch_bounds__(AP ? 512 : 256, AP ? 1 : BP_MIN_CTAS) k_block_pass(Geom g, TileMap tm, IndexPtrs ip, PassArgs a, BPGeom G) {
  if (rt_stopped(g.stop)) return;
  extern __shared__ __align__(128) unsigned char bp_smem[];
  __shared__ unsigned long long bars[4];
  __shared__ double red[16];
  __shared__ bool am_last;
  const int tid = threadIdx.x;
  const double zeta_v = a.zetap ? __ldg(a.zetap) : a.zeta;
  // GP: the core's tiles; AP: the fiber blocks' tiles; else every tile
  const i64 tfirst = AP ? tm.first[1] : 0;
  const i64 ntiles = (GP ? tm.first[1] : tm.first[tm.nblk]) - tfirst;
  const int esz = a.dtype == 0 ? 8 : 4;
  int* rmap = reinterpret_cast<int*>(bp_smem);
  double* gp = reinterpret_cast<double*>(bp_smem + (((size_t)G.rowmap_ints * 4 + 15) & ~(size_t)15));
  double* Asm = gp + G.gp_doubles;
  double* Aem = Asm + G.a_doubles;
  unsigned char* stage0 = reinterpret_cast<unsigned char*>(Aem + G.a_doubles);
  const size_t stage_bytes = (size_t)G.x_bytes + 2 * (size_t)G.w_doubles * 8;
  const char* xbase = reinterpret_cast<const char*>(a.xb);
  if (tid == 0) {
    for (int st = 0; st < G.stages; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tile t -> block b, first column q0 and column count (no divisions: tiles are cpt[b] whole columns)
  auto tile_cols = [&](i64 t, int& b, i64& q0, int& nc) {
    b = tile_block(tm, t);
    q0 = (t - tm.first[b]) * tm.cpt[b];
    nc = (int)min((i64)tm.cpt[b], g.blk[b].Q - q0);
  };
  // bulk-copy tile t (x range and, when used, the columns' W rows of both states)
  auto issue = [&](i64 t, int st) {
    int b, nc;
    i64 q0;
    tile_cols(t, b, q0, nc);
    const BlockDesc& bd = g.blk[b];
    unsigned char* sb = stage0 + (size_t)st * stage_bytes;
    const i64 e0 = q0 * bd.P, e1 = e0 + (i64)nc * bd.P;
    const i64 x0 = ((bd.off + e0) * esz) & ~(i64)15, x1 = ((bd.off + e1) * esz + 15) & ~(i64)15;
    const i64 q1 = q0 + nc;
    const i64 w0 = ((bd.w_off + q0 * bd.r) * 8) & ~(i64)15, w1 = ((bd.w_off + q1 * bd.r) * 8 + 15) & ~(i64)15;
    unsigned total = (unsigned)(x1 - x0);
    if (HS) total += (unsigned)(w1 - w0);
    if (HE) total += (unsigned)(w1 - w0);
    if (AP) total += (unsigned)((((q1 * bd.r) * 8 + 15) & ~(i64)15) - (((q0 * bd.r) * 8) & ~(i64)15));
    mbar_expect_tx(&bars[st], total);
    tma_load_1d(sb, xbase + x0, (unsigned)(x1 - x0), &bars[st]);
    if (HS) tma_load_1d(sb + G.x_bytes, reinterpret_cast<const char*>(a.st_s) + w0, (unsigned)(w1 - w0), &bars[st]);
    if (HE)
      tma_load_1d(sb + G.x_bytes + (size_t)G.w_doubles * 8, reinterpret_cast<const char*>(a.st_e) + w0,
                  (unsigned)(w1 - w0), &bars[st]);
    if (AP) {   // the columns' V rows in the second W slot (same 16-byte phase as W: w_off is 32-aligned)
      const i64 v0 = ((q0 * bd.r) * 8) & ~(i64)15, v1 = ((q1 * bd.r) * 8 + 15) & ~(i64)15;
      tma_load_1d(sb + G.x_bytes + (size_t)G.w_doubles * 8, reinterpret_cast<const char*>(a.V[bd.mode]) + v0,
                  (unsigned)(v1 - v0), &bars[st]);
    }
  };
  // contiguous tile range per CTA: at most a couple of block switches
  const i64 t_begin = tfirst + ntiles * blockIdx.x / gridDim.x, t_end = tfirst + ntiles * (blockIdx.x + 1) / gridDim.x;
  const i64 my_n = t_end - t_begin;
  if (tid == 0)
    for (int st = 0; st < G.stages && st < my_n; ++st) issue(t_begin + st, st);

  int cur_b = -1;
  double e2 = 0.0, x2 = 0.0;
  bool bad = false;
  double* acc = gp;   // AP: the block's partial A rows (P x r), zeroed at every block switch
  auto ap_flush = [&](int b) {
    __syncthreads();
    const i64 nout = g.blk[b].P * g.blk[b].r;
    double* dst = a.apart + ap_slot(g, tm, (int)gridDim.x, b, blockIdx.x);
    for (i64 o = tid; o < nout; o += blockDim.x) dst[o] = acc[o];
  };
  auto flush = [&](int b) {
    if (AP) {
      ap_flush(b);
      return;
    }
    const double se = block_sum(e2, red);
    const double sx = block_sum(x2, red);
    if (tid == 0 && a.partial) {
      a.partial[((i64)blockIdx.x * tm.nblk + b) * 2] = se;
      a.partial[((i64)blockIdx.x * tm.nblk + b) * 2 + 1] = sx;
    }
    e2 = 0.0;
    x2 = 0.0;
  };
  if (a.partial && tid < tm.nblk * 2) a.partial[(i64)blockIdx.x * tm.nblk * 2 + tid] = 0.0;
  int st = 0;
  unsigned phase = 0;
  for (i64 i = 0; i < my_n; ++i) {
    const i64 t = t_begin + i;
    int b, nc;
    i64 q0;
    tile_cols(t, b, q0, nc);
    const BlockDesc& bd = g.blk[b];
    const int P = (int)bd.P;
    const bool core = bd.is_core;
    const int r = bd.r;
    if (b != cur_b) {
      if (cur_b >= 0) flush(cur_b);   // (block_sum has barriers: everyone is done with the old row map)
      cur_b = b;
      if (WM && !core)
        for (int pp = tid; pp < P; pp += blockDim.x) rmap[pp] = ip.rowpos[bd.mode][pp];
      if (AP) {
        __syncthreads();   // the previous block's flush has read acc
        for (i64 o = tid; o < (i64)P * r; o += blockDim.x) acc[o] = 0.0;
      }
      if (tm.cols[b] && !AP) {   // lanes over columns: the block's A rows, row-major with an even pitch
        const int ap = (r + 1) & ~1;
        const i64 d = g.dim[bd.mode];
        for (int e = tid; e < P * ap; e += blockDim.x) {
          const int pp = e / ap, kk = e - pp * ap;
          const i64 row = core ? (i64)ip.rows[0][pp] : (i64)pp;
          if (HS) Asm[e] = kk < r ? a.st_s[g.a_off[bd.mode] + row + kk * d] : 0.0;
          if (HE) Aem[e] = kk < r ? a.st_e[g.a_off[bd.mode] + row + kk * d] : 0.0;
          if (GP) Aem[e] = kk < r ? a.U[(i64)pp * r + kk] : 0.0;   // U~_1 rows (the error state is unused)
        }
      }
      __syncthreads();
    }
    const unsigned char* sb = stage0 + (size_t)st * stage_bytes;
    const i64 e0 = q0 * P;
    const int xskip = (int)((((bd.off + e0) * esz) & 15) >> (esz == 8 ? 3 : 2));
    const int wskip = (int)((bd.w_off + q0 * r) & 1);
    BPTile T;
    T.x = sb + (size_t)xskip * esz;
    T.dtype = a.dtype;
    T.P = P;
    T.ncols = nc;
    T.r = r;
    T.As = HS ? a.st_s + g.a_off[bd.mode] : nullptr;
    T.Ae = HE ? a.st_e + g.a_off[bd.mode] : nullptr;
    T.d = g.dim[bd.mode];
    T.rows0 = core ? ip.rows[0] : nullptr;
    T.Wss = reinterpret_cast<const double*>(sb + G.x_bytes) + wskip;
    T.Wes = reinterpret_cast<const double*>(sb + G.x_bytes + (size_t)G.w_doubles * 8) + wskip;
    T.rmap = rmap;
    T.Asm = Asm;
    T.Aem = Aem;
    T.apitch = (r + 1) & ~1;
    T.Mk = (WM && !core) ? a.M[bd.mode] + q0 * g.nrows[bd.mode] : nullptr;
    T.mrows = (int)g.nrows[bd.mode];
    T.zeta = zeta_v;
    const i64 gofs = bd.off + e0;
    T.s_out = EXP && a.s_out ? a.s_out + gofs : nullptr;
    T.c_out = EXP && a.c_out ? a.c_out + gofs : nullptr;
    T.l_out = EXP && a.l_out ? a.l_out + gofs : nullptr;
    T.U = GP ? a.U : nullptr;
    T.t1 = GP ? a.t1 + q0 * r : nullptr;
    T.gp = gp;
    mbar_wait(&bars[st], phase);
    if (AP) bp_tile_ap<RB, HS>(T, acc);
    else if (core) bp_tile_r<RB, HS, HE, false, EXP, GP>(T, tm.cols[b] != 0, e2, x2, bad);
    else bp_tile_r<RB, HS, HE, WM, EXP, false>(T, tm.cols[b] != 0, e2, x2, bad);
    __syncthreads();   // stage st fully consumed
    if (tid == 0 && i + G.stages < my_n) issue(t_begin + i + G.stages, st);
    if (++st == G.stages) {
      st = 0;
      phase ^= 1u;
    }
  }
  if (cur_b >= 0) flush(cur_b);
  if (AP) return;
  if (bad) atomicExch(a.nonfinite, 1);
  if (a.partial == nullptr) return;
  if (tid == 0) {
    __threadfence();
    unsigned int ticket = atomicAdd(a.counter, 1u);
    am_last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // last CTA: per-block sums over CTAs in CTA order (deterministic)
  for (int bb = 0; bb < tm.nblk; ++bb) {
    if (tm.first[bb + 1] == tm.first[bb]) continue;   // block handled by the fiber pass (k_fiber.cuh)
    double se = 0.0, sx = 0.0;
    for (i64 c = tid; c < gridDim.x; c += blockDim.x) {
      se += ((volatile double*)a.partial)[(c * tm.nblk + bb) * 2];
      sx += ((volatile double*)a.partial)[(c * tm.nblk + bb) * 2 + 1];
    }
    se = block_sum(se, red);
    sx = block_sum(sx, red);
    if (tid == 0) {
      a.sums[2 * bb] = se;
      a.sums[2 * bb + 1] = sx;
    }
  }
  if (tid == 0) *a.counter = 0u;
}


