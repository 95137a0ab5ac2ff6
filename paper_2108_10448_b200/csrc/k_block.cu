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
#include "bp_types.cuh"

// ------------------------------------------------------------------ index prep

// rowpos_k[p] = position of p in the sorted row set I_k, or -1.
__device__ __forceinline__ void rowpos_mode(const Geom& g, const IndexPtrs& ip, int* __restrict__ rowpos_base, int k,
                                            i64 t0, i64 tstride) {
  i64 base = 0;
  for (int m = 0; m < k; ++m) base += g.dim[m];
  int* out = rowpos_base + base;
  const int* rows = ip.rows[k];
  const int nr = (int)g.nrows[k];
  for (i64 p = t0; p < g.dim[k]; p += tstride) {
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

__global__ void k_rowpos(Geom g, IndexPtrs ip, int* __restrict__ rowpos_base) {
  const int k = blockIdx.y;
  if (k >= g.n) return;
  rowpos_mode(g, ip, rowpos_base, k, blockIdx.x * (i64)blockDim.x + threadIdx.x, (i64)gridDim.x * blockDim.x);
}

// Per block column: the "rest" offset R over modes >= 2 and, for fiber blocks
// of modes >= 2, the fixed mode-1 index.  Mirrors tensor.py:250-283
// (decode_fiber_columns / fiber_base_offsets: other modes ascending, first
// other mode fastest) and, for the core, the np.ix_ ordering of tensor.py:239.
__device__ __forceinline__ void colprep_block(const Geom& g, const IndexPtrs& ip, i64* __restrict__ colR_base,
                                              int* __restrict__ coli1_base, const i64* __restrict__ col_off, int b,
                                              i64 t0, i64 tstride) {
  const BlockDesc bd = g.blk[b];
  i64* colR = colR_base + col_off[b];
  int* coli1 = coli1_base + col_off[b];
  for (i64 q = t0; q < bd.Q; q += tstride) {
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

__global__ void k_colprep(Geom g, IndexPtrs ip, i64* __restrict__ colR_base, int* __restrict__ coli1_base,
                          const i64* __restrict__ col_off) {
  const int b = blockIdx.y;
  if (b >= g.nblk) return;
  colprep_block(g, ip, colR_base, coli1_base, col_off, b, blockIdx.x * (i64)blockDim.x + threadIdx.x,
                (i64)gridDim.x * blockDim.x);
}

// Both index preparations in one launch: grid rows y < n are k_rowpos's modes,
// the rest k_colprep's blocks.
__global__ void k_prep(Geom g, IndexPtrs ip, int* __restrict__ rowpos_base, i64* __restrict__ colR_base,
                       int* __restrict__ coli1_base, const i64* __restrict__ col_off) {
  const int y = blockIdx.y;
  const i64 t0 = blockIdx.x * (i64)blockDim.x + threadIdx.x, ts = (i64)gridDim.x * blockDim.x;
  if (y < g.n) rowpos_mode(g, ip, rowpos_base, y, t0, ts);
  else if (y - g.n < g.nblk) colprep_block(g, ip, colR_base, coli1_base, col_off, y - g.n, t0, ts);
}

// ------------------------------------------------------------------ gather (sharded)

// x_b[e] = X_local[(i1 - lo) + (hi - lo) * R] when lo <= i1 < hi, else 0.
// With one rank (lo = 0, hi = d_1) this is the plain gather of solver.py:172-182.
// Multi-rank: every sampled entry has exactly one owner, so a sum all-reduce of
// the per-rank x_b reproduces the full gather bit-exactly.
// Optional copies of X with mode k fastest (mode k, then the other modes in order):
// fiber column j of mode k is then the contiguous run [d_k j, d_k (j + 1)).
struct ModeCopies {
  const void* p[RT_MAX_MODES];
};

__global__ void __launch_bounds__(256) k_gather(Geom g, TileMap tm, IndexPtrs ip, const void* __restrict__ X, int dtype,
                                               i64 lo, i64 hi, void* __restrict__ xb, ModeCopies mc) {
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
  const void* cp = (!core && bd.mode >= 1) ? mc.p[bd.mode] : nullptr;
  if (cp) {   // contiguous fibers from the mode-k-fastest copy (unsharded runs only)
    const i64* __restrict__ cols = ip.cols[bd.mode];
    for (i64 base = e0 + threadIdx.x; base < e1; base += (i64)GATHER_U * blockDim.x) {
      double v[GATHER_U];
#pragma unroll
      for (int u = 0; u < GATHER_U; ++u) {
        const i64 e = base + (i64)u * blockDim.x;
        v[u] = 0.0;
        if (e < e1) {
          i64 q, p;
          split_pq(e, P, small, q, p);
          v[u] = ld_elem(cp, p + P * cols[q], dtype);
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
    return;
  }
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

// Contiguous fiber columns (mode 1 of an unsharded X, or a mode-k-fastest copy):
// one warp per column, 16-byte vector copy into the compact block, plus the
// column's intersection rows X(I_k, q) into the fiber pass's copy (k_fiber.cuh).
// Core columns (unsharded X): the warp picks the rows I_1 out of the column's
// mode-1 fiber (one index load per entry, no per-entry division).
struct FastGather {
  const void* src[RT_MAX_MODES];   // mode 0: X (unsharded); k >= 1: the mode-k copy
  void* xi;
  i64 xi_off[RT_MAX_MODES], xi_ld[RT_MAX_MODES];
  unsigned ximask;                 // blocks whose intersection copy is written
  int nb;                          // blocks copied here
  int blk[RT_MAX_BLOCKS];
  i64 colbase[RT_MAX_BLOCKS + 1];  // prefix sums of their column counts
};

template <typename T>
__global__ void __launch_bounds__(256) k_gather_fibers(Geom g, IndexPtrs ip, FastGather fg, void* __restrict__ xb) {
  constexpr int VE = 16 / (int)sizeof(T);
  const int lane = threadIdx.x & 31;
  const i64 total = fg.colbase[fg.nb];
  for (i64 wc = blockIdx.x * (i64)(blockDim.x >> 5) + (threadIdx.x >> 5); wc < total;
       wc += (i64)gridDim.x * (blockDim.x >> 5)) {
    int f = 0;
    while (f + 1 < fg.nb && wc >= fg.colbase[f + 1]) ++f;
    const int b = fg.blk[f];
    const i64 q = wc - fg.colbase[f];
    const BlockDesc& bd = g.blk[b];
    const int k = bd.mode;
    const i64 P = bd.P;
    T* d = reinterpret_cast<T*>(xb) + bd.off + q * P;
    if (bd.is_core) {   // core column: rows I_1 of the mode-1 fiber X(:, i_2..i_n)
      const T* s = reinterpret_cast<const T*>(fg.src[0]) + g.dim[0] * ip.colR[0][q];
      const int* rows = ip.rows[0];
      for (i64 i = lane; i < P; i += 32) d[i] = __ldg(s + __ldg(rows + i));
      continue;
    }
    const T* s = reinterpret_cast<const T*>(fg.src[k]) + P * (k == 0 ? ip.colR[b][q] : ip.cols[k][q]);
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0 && P % VE == 0) {
      const float4* __restrict__ s4 = reinterpret_cast<const float4*>(s);
      float4* __restrict__ d4 = reinterpret_cast<float4*>(d);
      const i64 n4 = P / VE;
      // chunks of 8 vectors per lane: all loads in flight before the stores
      for (i64 base = 0; base < n4; base += 256) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const i64 i = base + u * 32 + lane;
          if (i < n4) v[u] = __ldg(s4 + i);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const i64 i = base + u * 32 + lane;
          if (i < n4) d4[i] = v[u];
        }
      }
    } else {
      for (i64 i = lane; i < P; i += 32) d[i] = __ldg(s + i);
    }
    if (fg.ximask >> b & 1) {
      const i64 ld = fg.xi_ld[k], nr = g.nrows[k];
      T* xo = reinterpret_cast<T*>(fg.xi) + fg.xi_off[k] + q * ld;
      const int* rows = ip.rows[k];
      for (i64 i = lane; i < ld; i += 32) xo[i] = i < nr ? __ldg(s + __ldg(rows + i)) : (T)0;
    }
  }
}

// Core block of an unsharded X: column q is X(I_1, i_2(q), .., i_n(q)), the rows
// I_1 of one mode-1 fiber.  I_1 is staged in shared memory once per CTA; a warp
// takes CW consecutive columns at a time and issues all their loads before the
// stores (the fiber's sectors are shared by the ~|I_1|/d_1 of it that is sampled).
#define GC_CW 4
template <typename T>
__global__ void __launch_bounds__(256) k_gather_core(Geom g, IndexPtrs ip, const void* __restrict__ X,
                                                     void* __restrict__ xb) {
  extern __shared__ int rows_s[];
  const BlockDesc& bd = g.blk[0];
  const int P = (int)bd.P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) rows_s[i] = ip.rows[0][i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const i64 Q = bd.Q, d1 = g.dim[0];
  const T* Xt = reinterpret_cast<const T*>(X);
  T* out = reinterpret_cast<T*>(xb) + bd.off;
  const i64* colR = ip.colR[0];
  constexpr int MAXR = 8;   // rows per lane held in flight per column (P <= 256 here)
  for (i64 q0 = (blockIdx.x * (i64)(blockDim.x >> 5) + (threadIdx.x >> 5)) * GC_CW; q0 < Q;
       q0 += (i64)gridDim.x * (blockDim.x >> 5) * GC_CW) {
    T v[GC_CW][MAXR];
#pragma unroll
    for (int c = 0; c < GC_CW; ++c) {
      const i64 q = q0 + c;
      if (q >= Q) break;
      const T* s = Xt + d1 * __ldg(colR + q);
#pragma unroll
      for (int u = 0; u < MAXR; ++u) {
        const int p = lane + 32 * u;
        if (p < P) v[c][u] = __ldg(s + rows_s[p]);
      }
    }
#pragma unroll
    for (int c = 0; c < GC_CW; ++c) {
      const i64 q = q0 + c;
      if (q >= Q) break;
      T* d = out + q * P;
#pragma unroll
      for (int u = 0; u < MAXR; ++u) {
        const int p = lane + 32 * u;
        if (p < P) d[p] = v[c][u];
      }
    }
  }
}

// out = X with mode k moved first: view X as (A, d_k, B) (A = prod_{m<k} d_m),
// out[i + d_k (a + A b)] = X[a + A (i + d_k b)] -- 32 x 32 shared-memory tiles,
// both sides coalesced.
template <typename T>
__global__ void __launch_bounds__(256) k_transpose_mode(const T* __restrict__ X, i64 A, i64 dk, i64 B,
                                                        T* __restrict__ out) {
  __shared__ T tile[32][33];
  const i64 a0 = (i64)blockIdx.x * 32, i0 = (i64)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  for (i64 b = blockIdx.z; b < B; b += gridDim.z) {
    const T* src = X + A * dk * b;
    T* dst = out + dk * A * b;
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
      const i64 a = a0 + tx, i = i0 + ty + r;
      if (a < A && i < dk) tile[ty + r][tx] = src[a + A * i];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
      const i64 i = i0 + tx, a = a0 + ty + r;
      if (a < A && i < dk) dst[i + dk * a] = tile[tx][ty + r];
    }
    __syncthreads();
  }
}

// K1 block pass (definition: bp_pass.cuh, instantiated in bp_rb*.cu)
template <bool HS, bool HE, bool WM, bool EXP, bool GP, int RB, bool AP>
__global__ void k_block_pass(Geom g, TileMap tm, IndexPtrs ip, PassArgs a, BPGeom G);

// A_k[p, a] = siginv_a * sum over the CTAs that touched block k+1 (CTA order) of the
// A-pass partials.  One thread per output (consecutive outputs, consecutive partials).
__global__ void __launch_bounds__(256) k_areduce_bp(Geom g, TileMap tm, PassArgs a, double* __restrict__ st_out) {
  if (rt_stopped(g.stop)) return;
  const int b = blockIdx.y + 1;
  if (b >= g.nblk || tm.first[b + 1] == tm.first[b]) return;   // (no tiles: the fiber pass writes A_k)
  const BlockDesc& bd = g.blk[b];
  const i64 N = tm.first[tm.nblk] - tm.first[1];
  const i64 G = a.ap_grid;
  const i64 c0 = ap_cta_of(tm.first[b] - tm.first[1], N, G), c1 = ap_cta_of(tm.first[b + 1] - 1 - tm.first[1], N, G);
  const i64 base = ap_slot(g, tm, (int)G, b, c0);
  const i64 nout = bd.P * bd.r, stride = nout;
  double* A = st_out + g.a_off[bd.mode];
  for (i64 o = blockIdx.x * (i64)blockDim.x + threadIdx.x; o < nout; o += (i64)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (i64 c = c0; c <= c1; ++c) s += a.apart[base + (c - c0) * stride + o];
    const i64 p = o / bd.r;
    const int aa = (int)(o - p * bd.r);
    A[p + (i64)aa * bd.P] = s * a.siginv[bd.mode][aa];
  }
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
