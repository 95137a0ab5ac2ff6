// k_block.cu -- index preparation, fused gather, the fused residual/threshold
// block pass (K1) and the streaming abs-max scan (K0).
//
// K1 replaces, per sampled entry, the reference's
//   _eval_blocks (solver.py:242-249 -> fiber_cur.py:288-326, the einsum hot spot)
//   hard_threshold(x_b - l_b, zeta) (solver.py:336-341 -> _core.pyx:252-262)
//   clean = x_b - s_b and the intersection extraction fib[rows-1, :] (fiber_cur.py:265)
//   sampled_relative_error sums (solver.py:209-231)
// in one pass over the compact sampled blocks: the low-rank value is evaluated
// on the fly from the rank-(r_1..r_n) Tucker state (G, A_k, W_b), so the
// reference's |J_k| * prod|I_m| einsum becomes r FMAs per entry.
#include "common.cuh"

// ------------------------------------------------------------------ index prep

// rowpos_k[p] = position of p in the sorted row set I_k, or -1.
__global__ void k_rowpos(Geom g, IndexPtrs ip, int* __restrict__ rowpos_base) {
  const int k = blockIdx.y;
  if (k >= g.n) return;
  i64 base = 0;
  for (int m = 0; m < k; ++m) base += g.dim[m];
  int* out = rowpos_base + base;
  const int* rows = ip.rows[k];
  const int nr = (int)g.nrows[k];
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < g.dim[k]; p += (i64)gridDim.x * blockDim.x) {
    int lo = 0, hi = nr - 1, pos = -1;
    while (lo <= hi) {
      int mid = (lo + hi) >> 1;
      int v = rows[mid];
      if (v == (int)p) { pos = mid; break; }
      if (v < (int)p) lo = mid + 1; else hi = mid - 1;
    }
    out[p] = pos;
  }
}

// Per block column: the "rest" offset R over modes >= 2 and, for fiber blocks
// of modes >= 2, the fixed mode-1 index.  Mirrors tensor.py:250-283
// (decode_fiber_columns / fiber_base_offsets: other modes ascending, first
// other mode fastest) and, for the core, the np.ix_ ordering of tensor.py:239.
__global__ void k_colprep(Geom g, IndexPtrs ip, i64* __restrict__ colR_base, int* __restrict__ coli1_base,
                          const i64* __restrict__ col_off) {
  const int b = blockIdx.y;
  if (b >= g.nblk) return;
  const BlockDesc bd = g.blk[b];
  i64* colR = colR_base + col_off[b];
  int* coli1 = coli1_base + col_off[b];
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < bd.Q; q += (i64)gridDim.x * blockDim.x) {
    i64 R = 0;
    int i1 = -1;
    if (bd.is_core) {
      i64 t = q;
      for (int m = 1; m < g.n; ++m) {
        i64 pos = t % g.nrows[m];
        t /= g.nrows[m];
        R += (i64)ip.rows[m][pos] * g.rstride[m];
      }
    } else {
      const int k = bd.mode;
      i64 j = ip.cols[k][q];
      for (int m = 0; m < g.n; ++m) {
        if (m == k) continue;
        i64 im = j % g.dim[m];
        j /= g.dim[m];
        if (m == 0) i1 = (int)im; else R += im * g.rstride[m];
      }
    }
    colR[q] = R;
    coli1[q] = i1;
  }
}

// ------------------------------------------------------------------ tile map

#define GATHER_U 4
#define PASS_U 4
#define TILE_MAX_ELEMS 4096

struct TileMap {
  int nblk;
  int tile;                        // max elements per tile
  i64 first[RT_MAX_BLOCKS + 1];    // first tile of each block, first[nblk] = total tiles
  i64 te[RT_MAX_BLOCKS];           // elements per tile of each block (whole columns when P <= tile)
};

// (q, p) = divmod(e, P) -- 32-bit when the block fits (always for the BASELINE shapes)
__device__ __forceinline__ void split_pq(i64 e, i64 P, bool small, i64& q, i64& p) {
  if (small) {
    const unsigned int qq = (unsigned int)e / (unsigned int)P;
    q = qq;
    p = (i64)((unsigned int)e - qq * (unsigned int)P);
  } else {
    q = e / P;
    p = e - q * P;
  }
}

__device__ __forceinline__ int tile_block(const TileMap& tm, i64 t) {
  int b = 0;
  while (b + 1 < tm.nblk && t >= tm.first[b + 1]) ++b;
  return b;
}

// ------------------------------------------------------------------ gather (sharded)

// x_b[e] = X_local[(i1 - lo) + (hi - lo) * R] when lo <= i1 < hi, else 0.
// With one rank (lo = 0, hi = d_1) this is the plain gather of solver.py:172-182.
// Multi-rank: every sampled entry has exactly one owner, so a sum all-reduce of
// the per-rank x_b reproduces the full gather bit-exactly.
__global__ void __launch_bounds__(256) k_gather(Geom g, TileMap tm, IndexPtrs ip, const void* __restrict__ X, int dtype,
                                               i64 lo, i64 hi, void* __restrict__ xb) {
  const i64 t = blockIdx.x;
  const int b = tile_block(tm, t);
  const BlockDesc& bd = g.blk[b];
  const i64 P = bd.P;
  const i64 nel = P * bd.Q;
  const i64 e0 = (t - tm.first[b]) * tm.te[b];
  const i64 e1 = min(nel, e0 + tm.te[b]);
  const i64 ld = hi - lo;
  const i64* __restrict__ colR = ip.colR[b];
  const int* __restrict__ coli1 = ip.coli1[b];
  const int* __restrict__ rows0 = ip.rows[0];
  const bool core = bd.is_core;
  const i64 rstr = bd.mode >= 1 ? g.rstride[bd.mode] : 0;
  const i64 off = bd.off;
  const bool small = nel < 0xFFFFFFFFll;
  for (i64 base = e0 + threadIdx.x; base < e1; base += (i64)GATHER_U * blockDim.x) {
    double v[GATHER_U];
#pragma unroll
    for (int u = 0; u < GATHER_U; ++u) {
      const i64 e = base + (i64)u * blockDim.x;
      v[u] = 0.0;
      if (e < e1) {
        i64 q, p;
        split_pq(e, P, small, q, p);
        const int ci = coli1[q];
        const i64 i1 = ci >= 0 ? (i64)ci : (core ? (i64)rows0[p] : p);
        if (i1 >= lo && i1 < hi) v[u] = ld_elem(X, (i1 - lo) + ld * (colR[q] + p * rstr), dtype);
      }
    }
#pragma unroll
    for (int u = 0; u < GATHER_U; ++u) {
      const i64 e = base + (i64)u * blockDim.x;
      if (e < e1) {
        if (dtype == 0) reinterpret_cast<double*>(xb)[off + e] = v[u];
        else reinterpret_cast<float*>(xb)[off + e] = (float)v[u];
      }
    }
  }
}

// ------------------------------------------------------------------ K1 block pass

struct PassArgs {
  const void* xb;
  int dtype;
  const double* st_s;      // state giving L for the threshold (null: L = 0, first iteration)
  const double* st_e;      // state giving L for the error / trace (null: no error)
  double zeta;
  double* M[RT_MAX_MODES]; // intersection outputs, m_k x p_k column-major (null: skip)
  double* s_out;           // optional sparse values on the blocks
  double* c_out;           // optional clean values
  double* l_out;           // optional low-rank values (state st_e)
  double* partial;         // [tiles][2] per-CTA (e2, x2)
  double* sums;            // [nblk][2]  final (e2, x2)
  unsigned int* counter;   // last-CTA ticket
  int* nonfinite;          // set if a clean intersection entry is not finite
  int want_x2;
};

// ---- TMA (cp.async.bulk) + mbarrier helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Shared-memory geometry of the persistent block pass (computed on the host).
struct BPGeom {
  int stages;
  int x_bytes;       // x region per stage (bytes, >= tile bytes + 16)
  int w_doubles;     // W region per stage and state (doubles, >= cpt*r + 2)
  int a_doubles;     // A region per state (doubles, >= max block rows * rp); 0: A read from global
  int rowmap_ints;   // rowpos staging (ints, >= max fiber-block rows)
  int rp_max;
};

__host__ __device__ inline int bp_rp(int r) { return r | 1; }   // odd row pitch: conflict-free smem rows
__host__ __device__ inline long long bp_smem_bytes(const BPGeom& G) {
  const long long stage = (long long)G.x_bytes + 2LL * G.w_doubles * 8;
  return 2LL * G.a_doubles * 8 + (((long long)G.rowmap_ints * 4 + 15) & ~15LL) + (long long)G.stages * stage;
}

// Persistent K1 block pass.  CTA c processes tiles c, c + grid, ... of the
// compact blocks (tiles are whole columns of one block, so x and the
// columns' W rows are contiguous).  Each tile's x, W_s, W_e ranges are
// streamed into a shared-memory ring by cp.async.bulk (one mbarrier per
// stage).  At every block switch the block's A rows (both states, row pitch
// rp) and its intersection row map are staged into shared memory, so the
// per-entry work -- L = A[row] . W[col] (r FMAs per state), hard threshold,
// clean value, intersection scatter, error sums -- reads only shared memory.
// Per-(CTA, block) partial sums are combined by the last CTA in CTA order
// (deterministic: the tile -> CTA assignment is static).
// Per-tile inner loop, specialised on the exact rank R and the pass variant:
// HS = threshold state present (iteration >= 2), HE = error state present,
// WM = write the clean intersection rows, EXP = export outputs (s/c/l, runtime).
// All indices are tile-local 32-bit; operands come from shared memory.
// R = 0: runtime rank r.  GA: A read from global memory (column-major, stride d,
// core rows through rows0) when the staged copy does not fit shared memory.
template <int R, bool HS, bool HE, bool WM, bool EXP, bool GA>
__device__ __forceinline__ void bp_tile(const unsigned char* __restrict__ sb, int dtype, int xskip, int n, int e0, int P,
                                        int q0, const double* __restrict__ As, const double* __restrict__ Ae, int rp,
                                        const double* __restrict__ Wss, const double* __restrict__ Wes,
                                        const int* __restrict__ rmap, double* __restrict__ Mk, int mrows, double zeta,
                                        double* __restrict__ s_out, double* __restrict__ c_out,
                                        double* __restrict__ l_out, double& e2, double& x2, bool& bad, int r_rt,
                                        i64 d, const int* __restrict__ rows0) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int r = R > 0 ? R : r_rt;
  int q = (e0 + tid) / P, p = (e0 + tid) - q * P;
  const int dq = nt / P, dp = nt - dq * P;
  const double* xd = reinterpret_cast<const double*>(sb) + xskip;
  const float* xf = reinterpret_cast<const float*>(sb) + xskip;
  for (int k = tid; k < n; k += nt) {
    const double x = dtype == 0 ? xd[k] : (double)xf[k];
    const int ql = q - q0;
    double ls = 0.0;
    const i64 grow = GA ? (rows0 ? (i64)rows0[p] : (i64)p) : 0;
    if (HS) {
      const double* wr = Wss + ql * r;
      if (GA) {
        const double* ar = As + grow;
        if (R > 0) {
#pragma unroll
          for (int kk = 0; kk < (R > 0 ? R : 1); ++kk) ls = fma(ar[kk * d], wr[kk], ls);
        } else {
          for (int kk = 0; kk < r; ++kk) ls = fma(ar[kk * d], wr[kk], ls);
        }
      } else {
        const double* ar = As + p * rp;
        if (R > 0) {
#pragma unroll
          for (int kk = 0; kk < (R > 0 ? R : 1); ++kk) ls = fma(ar[kk], wr[kk], ls);
        } else {
          for (int kk = 0; kk < r; ++kk) ls = fma(ar[kk], wr[kk], ls);
        }
      }
    }
    const double sv = fabs(x - ls) <= zeta ? 0.0 : x - ls;
    const double c = x - sv;
    if (WM) {
      const int pos = rmap[p];
      if (pos >= 0) {
        Mk[pos + q * mrows] = c;
        bad |= !isfinite(c);
      }
    }
    double le = 0.0;
    if (HE) {
      const double* wr = Wes + ql * r;
      if (GA) {
        const double* ar = Ae + grow;
        if (R > 0) {
#pragma unroll
          for (int kk = 0; kk < (R > 0 ? R : 1); ++kk) le = fma(ar[kk * d], wr[kk], le);
        } else {
          for (int kk = 0; kk < r; ++kk) le = fma(ar[kk * d], wr[kk], le);
        }
      } else {
        const double* ar = Ae + p * rp;
        if (R > 0) {
#pragma unroll
          for (int kk = 0; kk < (R > 0 ? R : 1); ++kk) le = fma(ar[kk], wr[kk], le);
        } else {
          for (int kk = 0; kk < r; ++kk) le = fma(ar[kk], wr[kk], le);
        }
      }
      const double rr = x - le - sv;
      e2 = fma(rr, rr, e2);
    }
    if (EXP) {
      if (s_out) s_out[k] = sv;
      if (c_out) c_out[k] = c;
      if (l_out) l_out[k] = le;
    }
    x2 = fma(x, x, x2);
    p += dp;
    q += dq;
    if (p >= P) { p -= P; ++q; }
  }
}

template <bool HS, bool HE, bool WM, bool EXP>
__device__ __forceinline__ void bp_tile_r(int r, bool ga, const unsigned char* sb, int dtype, int xskip, int n, int P,
                                          const double* As, const double* Ae, int rp, const double* Wss,
                                          const double* Wes, const int* rmap, double* Mk, int mrows, double zeta,
                                          double* s_out, double* c_out, double* l_out, double& e2, double& x2,
                                          bool& bad, i64 d, const int* rows0) {
  if (ga) {
    bp_tile<0, HS, HE, WM, EXP, true>(sb, dtype, xskip, n, 0, P, 0, As, Ae, rp, Wss, Wes, rmap, Mk, mrows, zeta, s_out,
                                      c_out, l_out, e2, x2, bad, r, d, rows0);
    return;
  }
#define BP_CASE(RR)                                                                                                   \
  case RR:                                                                                                            \
    bp_tile<RR, HS, HE, WM, EXP, false>(sb, dtype, xskip, n, 0, P, 0, As, Ae, rp, Wss, Wes, rmap, Mk, mrows, zeta,   \
                                        s_out, c_out, l_out, e2, x2, bad, r, d, rows0);                               \
    break;
  switch (r) {
    BP_CASE(1) BP_CASE(2) BP_CASE(3) BP_CASE(4) BP_CASE(5) BP_CASE(6) BP_CASE(7) BP_CASE(8) BP_CASE(10) BP_CASE(12)
    BP_CASE(16)
    default:
      bp_tile<0, HS, HE, WM, EXP, false>(sb, dtype, xskip, n, 0, P, 0, As, Ae, rp, Wss, Wes, rmap, Mk, mrows, zeta,
                                         s_out, c_out, l_out, e2, x2, bad, r, d, rows0);
      break;
  }
#undef BP_CASE
}

// Persistent K1 block pass.  CTA c processes a contiguous range of tiles of
// the compact blocks (tiles are whole columns of one block, so x and the
// columns' W rows are contiguous).  Each tile's x, W_s, W_e ranges are
// streamed into a shared-memory ring by cp.async.bulk (one mbarrier per
// stage).  At every block switch the block's A rows (both states, row pitch
// rp) and its intersection row map are staged into shared memory, so the
// per-entry work -- L = A[row] . W[col] (r FMAs per state), hard threshold,
// clean value, intersection scatter, error sums -- reads only shared memory.
// Per-(CTA, block) partial sums are combined by the last CTA in CTA order
// (deterministic: the tile -> CTA assignment is static).
template <bool HS, bool HE, bool WM, bool EXP>
__global__ void __launch_bounds__(256) k_block_pass(Geom g, TileMap tm, IndexPtrs ip, PassArgs a, BPGeom G) {
  extern __shared__ __align__(128) unsigned char bp_smem[];
  __shared__ unsigned long long bars[4];
  __shared__ double red[8];
  __shared__ bool am_last;
  const int tid = threadIdx.x;
  const i64 ntiles = tm.first[tm.nblk];
  const int esz = a.dtype == 0 ? 8 : 4;
  double* A_s = reinterpret_cast<double*>(bp_smem);
  double* A_e = A_s + G.a_doubles;
  int* rmap = reinterpret_cast<int*>(A_e + G.a_doubles);
  unsigned char* stage0 = reinterpret_cast<unsigned char*>(rmap) + (((size_t)G.rowmap_ints * 4 + 15) & ~(size_t)15);
  const size_t stage_bytes = (size_t)G.x_bytes + 2 * (size_t)G.w_doubles * 8;
  const char* xbase = reinterpret_cast<const char*>(a.xb);
  if (tid == 0) {
    for (int st = 0; st < G.stages; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto tile_range = [&](i64 t, int& b, i64& e0, i64& e1) {
    b = tile_block(tm, t);
    const i64 nel = g.blk[b].P * g.blk[b].Q;
    e0 = (t - tm.first[b]) * tm.te[b];
    e1 = min(nel, e0 + tm.te[b]);
  };
  // bulk-copy tile t (x range and, when used, the columns' W rows of both states)
  auto issue = [&](i64 t, int st) {
    int b;
    i64 e0, e1;
    tile_range(t, b, e0, e1);
    const BlockDesc& bd = g.blk[b];
    unsigned char* sb = stage0 + (size_t)st * stage_bytes;
    const i64 x0 = ((bd.off + e0) * esz) & ~(i64)15, x1 = ((bd.off + e1) * esz + 15) & ~(i64)15;
    const i64 q0 = e0 / bd.P, q1 = (e1 + bd.P - 1) / bd.P;
    const i64 w0 = ((bd.w_off + q0 * bd.r) * 8) & ~(i64)15, w1 = ((bd.w_off + q1 * bd.r) * 8 + 15) & ~(i64)15;
    unsigned total = (unsigned)(x1 - x0);
    if (HS) total += (unsigned)(w1 - w0);
    if (HE) total += (unsigned)(w1 - w0);
    mbar_expect_tx(&bars[st], total);
    tma_load_1d(sb, xbase + x0, (unsigned)(x1 - x0), &bars[st]);
    if (HS) tma_load_1d(sb + G.x_bytes, reinterpret_cast<const char*>(a.st_s) + w0, (unsigned)(w1 - w0), &bars[st]);
    if (HE)
      tma_load_1d(sb + G.x_bytes + (size_t)G.w_doubles * 8, reinterpret_cast<const char*>(a.st_e) + w0,
                  (unsigned)(w1 - w0), &bars[st]);
  };
  // contiguous tile range per CTA: at most a couple of block switches (A staging)
  const i64 t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  const i64 my_n = t_end - t_begin;
  if (tid == 0)
    for (int st = 0; st < G.stages && st < my_n; ++st) issue(t_begin + st, st);

  int cur_b = -1;
  double e2 = 0.0, x2 = 0.0;
  bool bad = false;
  auto flush = [&](int b) {
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
  for (i64 i = 0; i < my_n; ++i) {
    const i64 t = t_begin + i;
    const int st = (int)(i % G.stages);
    int b;
    i64 e0, e1;
    tile_range(t, b, e0, e1);
    const BlockDesc& bd = g.blk[b];
    const int P = (int)bd.P;
    const bool core = bd.is_core;
    const int r = bd.r, rp = bp_rp(r);
    const bool a_sm = G.a_doubles > 0;
    if (b != cur_b) {
      if (cur_b >= 0) flush(cur_b);   // (block_sum has barriers: everyone is done with the old A)
      cur_b = b;
      __syncthreads();
      const i64 d = g.dim[bd.mode];
      const int* rows0 = ip.rows[0];
      if (a_sm)
        for (int e = tid; e < P * r; e += blockDim.x) {
          const int pp = e % P, kk = e / P;
          const i64 row = core ? (i64)rows0[pp] : pp;
          if (HS) A_s[pp * rp + kk] = a.st_s[g.a_off[bd.mode] + row + kk * d];
          if (HE) A_e[pp * rp + kk] = a.st_e[g.a_off[bd.mode] + row + kk * d];
        }
      if (WM && !core)
        for (int pp = tid; pp < P; pp += blockDim.x) rmap[pp] = ip.rowpos[bd.mode][pp];
      __syncthreads();
    }
    const unsigned char* sb = stage0 + (size_t)st * stage_bytes;
    const int xskip = (int)((((bd.off + e0) * esz) & 15) / esz);
    const i64 q0 = e0 / P;
    const int wskip = (int)((((bd.w_off + q0 * r) * 8) & 15) / 8);
    const double* Wss = reinterpret_cast<const double*>(sb + G.x_bytes) + wskip;
    const double* Wes = reinterpret_cast<const double*>(sb + G.x_bytes + (size_t)G.w_doubles * 8) + wskip;
    mbar_wait(&bars[st], (unsigned)((i / G.stages) & 1));
    const int n = (int)(e1 - e0);
    const i64 gofs = bd.off + e0;
    // tile-local indexing: q counts columns from the tile start (tiles are whole columns)
    const double* Ags = HS ? (a_sm ? A_s : a.st_s + g.a_off[bd.mode]) : nullptr;
    const double* Age = HE ? (a_sm ? A_e : a.st_e + g.a_off[bd.mode]) : nullptr;
    if (core) {
      bp_tile_r<HS, HE, false, EXP>(r, !a_sm, sb, a.dtype, xskip, n, P, Ags, Age, rp, Wss, Wes, rmap, nullptr, 0,
                                    a.zeta, EXP && a.s_out ? a.s_out + gofs : nullptr,
                                    EXP && a.c_out ? a.c_out + gofs : nullptr,
                                    EXP && a.l_out ? a.l_out + gofs : nullptr, e2, x2, bad, g.dim[bd.mode],
                                    ip.rows[0]);
    } else {
      bp_tile_r<HS, HE, WM, EXP>(r, !a_sm, sb, a.dtype, xskip, n, P, Ags, Age, rp, Wss, Wes, rmap,
                                 WM ? a.M[bd.mode] + q0 * g.nrows[bd.mode] : nullptr, (int)g.nrows[bd.mode], a.zeta,
                                 EXP && a.s_out ? a.s_out + gofs : nullptr, EXP && a.c_out ? a.c_out + gofs : nullptr,
                                 EXP && a.l_out ? a.l_out + gofs : nullptr, e2, x2, bad, g.dim[bd.mode], nullptr);
    }
    __syncthreads();   // stage st fully consumed
    if (tid == 0 && i + G.stages < my_n) issue(t_begin + i + G.stages, st);
  }
  if (cur_b >= 0) flush(cur_b);
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

// ------------------------------------------------------------------ K0 abs-max

// zeta_0 = max|X| (solver.py:184-192, used when cfg.zeta0 is None, solver.py:304).
// NaN propagates like numpy's max.  Result is written as the IEEE bit pattern
// of a nonnegative double (monotone as an unsigned integer) via atomicMax.
template <typename T>
__global__ void __launch_bounds__(256) k_absmax(const T* __restrict__ x, i64 n, unsigned long long* __restrict__ out) {
  __shared__ double red[8];
  double m = 0.0;
  bool nan = false;
  constexpr int VEC = 16 / sizeof(T);
  const i64 nv = n / VEC;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  // 4 independent 16-byte loads in flight per thread
  for (; i + 3 * stride < nv; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(xv + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const T* e = reinterpret_cast<const T*>(&v[u]);
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        double a = fabs((double)e[j]);
        nan |= (a != a);
        m = fmax(m, a);
      }
    }
  }
  for (; i < nv; i += stride) {
    uint4 v = __ldcs(xv + i);
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      double a = fabs((double)e[j]);
      nan |= (a != a);
      m = fmax(m, a);
    }
  }
  for (i64 j = nv * VEC + blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += stride) {
    double a = fabs((double)x[j]);
    nan |= (a != a);
    m = fmax(m, a);
  }
  m = block_max(m, red);
  int anynan = __syncthreads_or(nan);
  if (threadIdx.x == 0) {
    unsigned long long bits = anynan ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(m);
    atomicMax(out, bits);
  }
}

template __global__ void k_absmax<float>(const float*, i64, unsigned long long*);
template __global__ void k_absmax<double>(const double*, i64, unsigned long long*);

// ------------------------------------------------------------------ kernel-level plug

// gather_columns (reference _core.pyx:265-288): out[i, c] = flat[bases[c] + i*stride],
// out is length x ncols column-major (the Cython backend's F-order result).
__global__ void k_gather_columns(const void* __restrict__ flat, int dtype, const i64* __restrict__ bases, i64 ncols,
                                 i64 stride, i64 length, double* __restrict__ out) {
  const i64 n = ncols * length;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
    i64 c = e / length, i = e - c * length;
    out[e] = ld_elem(flat, bases[c] + i * stride, dtype);
  }
}

// hard_threshold (reference _core.pyx:252-262): strict keep |x| > zeta.
__global__ void k_hard_threshold(const double* __restrict__ a, i64 n, double zeta, double* __restrict__ out) {
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x)
    out[e] = hard_thr(a[e], zeta);
}
