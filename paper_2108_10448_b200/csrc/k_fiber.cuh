// k_fiber.cuh -- the K1 threshold and error passes over the fiber blocks,
// staged by TMA (template definition; instantiated per dtype in
// k_fiber_f32.cu / k_fiber_f64.cu so they compile in parallel).
//
// Per sampled fiber entry (p, q) of block k (mode-k fiber q of the compact
// sample, reference solver.py:336-355):
//   L_s = A_k^s[p, :] . W^s[q, :]       (previous iterate; 0 at iteration 1)
//   S   = HT(x - L_s, zeta)             strict |.| > zeta keep (py_kernels.py:226-230)
//   threshold pass: clean = x - S, written to the intersection M_k when p is in I_k
//                   (fiber_cur.py:265, fib[rows - 1, :])
//   error pass:     L_e = A_k^e[p, :] . W^e[q, :] (new iterate),
//                   sums of (x - L_e - S)^2 and x^2 (solver.py:209-231)
// The arithmetic per entry is the same sequence of fp64 operations as
// k_block_pass (bp_pass.cuh), so S, the clean values and M are bit-identical.
//
// Mapping (the K3 design, k_full_tma.cu): a CTA owns a band of H rows of a
// block and a contiguous run of column groups; each consumer thread owns V
// consecutive rows (one vector) with their A rows of both states in registers
// for the whole band and its intersection positions; a producer warp streams
// the group's x columns (one bulk copy when the band is the whole fiber) and
// the columns' W rows of both states into an NST-deep shared-memory ring
// (full/empty mbarriers).  Sums are per-(CTA, block) partials reduced by the
// last CTA in CTA order (deterministic).
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "bp_types.cuh"
#include "fiber_types.cuh"

#define FB_MAX_CONS 352   // + the producer warp: 12 warps, so up to 168 registers per thread
#define FB_STAGE_BYTES (32 * 1024)
#define FB_SMEM_BUDGET (100 * 1024)   // two CTAs per SM
#define FB_MAX_CTAS_PER_SM 2
#define FB_MAX_STAGES 8
#define FB_MAX_R 16
#ifndef FB_COL_UNROLL
#define FB_COL_UNROLL 1   // columns in flight per consumer thread (A/B: make EXTRA=-DFB_COL_UNROLL=2)
#endif

struct FiberBlk {
  i64 off;      // element offset of the block in its buffer
  i64 P, Q;     // rows (column stride) and columns (|J_k|)
  i64 dA;       // leading dimension of A_k (d_k)
  const int* amap;   // threshold pass over the intersection copy: row -> I_k row (A rows); null: identity
  int Pv;       // valid rows (|I_k| with amap, else P)
  i64 w_off;    // W rows of the block in a state
  i64 a_off;    // A_k in a state (d_k x r column-major)
  i64 tfirst;   // first tile of the block
  i64 ncg;      // column groups per band
  int nbands;
  int H, nchB, cpr, CB;
  int b, mode, r, mrows;
  i64 pbase;    // A pass: first partial slot of the block (doubles)
  int c0;       // A pass: first CTA whose tile range touches the block
};

struct FiberArgs {
  const int* stop;   // the engine's stop flag (iteration launches), or null
  const void* xb;
  const double* st_s;
  const double* st_e;
  double zeta;
  const double* zetap;
  double* M[RT_MAX_MODES];
  const int* rowpos[RT_MAX_MODES];
  double* partial;
  double* sums;
  unsigned int* counter;
  int* nonfinite;
  int nfb;        // handled blocks
  int nblk;       // all blocks (partial stride)
  int nst;
  int reserve_sms;   // (host: grid sizing)
  int x_region;   // bytes of x per stage
  int w_region;   // bytes of W rows per stage and state
  i64 ntiles;
  // A pass: A_k = C_k V_k Sigma_k^+ (fiber_cur.py:267, fib @ pinv) -- the clean fiber
  // entries times the staged V rows, per-(CTA, block) partial rows, reduced in CTA order
  const double* Vr[RT_MAX_MODES];       // |J_k| x r row-major
  const double* siginv[RT_MAX_MODES];
  double* apart;
  double* a_out;                        // state receiving A_k (d_k x r column-major at a_off)
  FiberBlk fb[RT_MAX_MODES];
};

template <typename T, int V>
struct alignas(V * sizeof(T)) FbVec {
  T v[V];
};

// elements per thread: the widest vector whose A rows (V * R per state) stay
// within 32 doubles of registers
template <typename T>
__host__ __device__ constexpr int fb_vec(int r, int ns) {
  return (int)(16 / sizeof(T)) * r * ns <= 48 ? (int)(16 / sizeof(T))
         : (int)(8 / sizeof(T)) * r * ns <= 48 ? (int)(8 / sizeof(T))
         : (int)(4 / sizeof(T)) >= 1 ? (int)(4 / sizeof(T)) : 1;
}

// scalar-row blocks (SC): rows per thread, loaded one element at a time (the columns
// are not vector-aligned) -- as many as keep the A rows within 48 doubles, so the
// column's W rows and the loop overhead are shared by up to four entries
__host__ __device__ constexpr int fb_sc_vec(int r, int ns) {
  return 4 * r * ns <= 48 ? 4 : 2 * r * ns <= 48 ? 2 : 1;
}

__device__ __forceinline__ void fb_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// sum over the consumer warps only (named barrier 1; the producer warp is elsewhere)
__device__ __forceinline__ double fb_cons_sum(double v, double* red, int ncons) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory");
  if (lane == 0) red[w] = v;
  asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory");
  double t = 0.0;
  for (int i = 0; i < (ncons >> 5); ++i) t += red[i];
  asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory");
  return t;
}

// ns_reg: doubles of per-row register state per rank (A rows of the states, A-pass accumulators)
template <bool HS, bool HE, bool AP>
__host__ __device__ constexpr int fb_nsreg() {
  return ((HS ? 1 : 0) + (HE ? 1 : 0) + (AP ? 1 : 0)) > 0 ? (HS ? 1 : 0) + (HE ? 1 : 0) + (AP ? 1 : 0) : 1;
}

// SC: scalar rows (fb_sc_vec per thread) for blocks whose columns are not 16-byte multiples (the
// core, |I_1| rows): whole-column tiles whose starts stay 16-byte aligned.
template <typename T, int R, bool EX, bool HS, bool HE, bool AP, bool SC>
__global__ void __launch_bounds__(FB_MAX_CONS + 32, 1) k_fiber_pass(FiberArgs a) {   // (grid: up to 2 CTAs per SM)
  if (rt_stopped(a.stop)) return;
  constexpr int NS = (HS ? 1 : 0) + ((HE || AP) ? 1 : 0);   // staged row sets per column: W_s, W_e or V
  constexpr int V = SC ? fb_sc_vec(R, fb_nsreg<HS, HE, AP>()) : fb_vec<T>(R, fb_nsreg<HS, HE, AP>());
  constexpr bool WM = !HE && !AP;   // threshold pass: intersections
  constexpr bool SUMS = HE;         // error pass: sums
  typedef FbVec<T, V> VT;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ double red[FB_MAX_CONS / 32 + 1];
  __shared__ double red2[FB_MAX_CONS / 32 + 1];
  __shared__ bool am_last;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm);
  unsigned long long* empty = full + FB_MAX_STAGES;
  unsigned char* ring = sm + 2 * FB_MAX_STAGES * 8;
  const int tid = threadIdx.x, lane = tid & 31;
  const int ncons = blockDim.x - 32;
  const i64 stage_bytes = (i64)a.x_region + (i64)NS * a.w_region;
  if (tid == 0) {
    for (int s = 0; s < a.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (SUMS && tid < a.nfb * 2) a.partial[((i64)blockIdx.x * a.nblk + a.fb[tid >> 1].b) * 2 + (tid & 1)] = 0.0;
  __syncthreads();
  const i64 t0 = a.ntiles * blockIdx.x / gridDim.x, t1 = a.ntiles * (blockIdx.x + 1) / gridDim.x;
  bool bad = false;
  // tile cursor: (handled block f, band, column group), advanced tile by tile (no divisions)
  int cf = 0;
  while (cf + 1 < a.nfb && t0 >= a.fb[cf + 1].tfirst) ++cf;
  i64 cband, ccg;
  {
    const i64 lt = t0 - a.fb[cf].tfirst;
    cband = lt / a.fb[cf].ncg;
    ccg = lt - cband * a.fb[cf].ncg;
  }
  auto advance = [&]() {
    if (++ccg == a.fb[cf].ncg) {
      ccg = 0;
      if (++cband == a.fb[cf].nbands) {
        cband = 0;
        ++cf;
      }
    }
  };
  if (tid >= ncons) {
    // ---------------- producer warp
    const char* xb = reinterpret_cast<const char*>(a.xb);
    int s = 0;
    unsigned ph = 0;
    for (i64 t = t0, k = 0; t < t1; ++t, ++k, advance()) {
      if (k >= a.nst) mbar_wait(&empty[s], ph ^ 1u);
      const FiberBlk& B = a.fb[cf];
      const i64 r0 = cband * B.H, hb = min((i64)B.H, B.P - r0);
      const i64 c0 = ccg * B.CB, nc = min((i64)B.CB, B.Q - c0);
      unsigned char* dst = ring + s * stage_bytes;
      const unsigned wbytes = (unsigned)((nc * B.r * 8 + 15) & ~15LL);
      const i64 wsrc = (B.w_off + c0 * B.r) * 8;
      if (lane == 0) {
        const unsigned xbytes = (unsigned)((hb * nc * (i64)sizeof(T) + 15) & ~15LL);   // (SC: rounded up)
        mbar_expect_tx(&full[s], xbytes + NS * wbytes);
        int slot = 0;
        if (HS) tma_load_1d(dst + a.x_region + (slot++) * a.w_region, reinterpret_cast<const char*>(a.st_s) + wsrc,
                            wbytes, &full[s]);
        if (HE) tma_load_1d(dst + a.x_region + slot * a.w_region, reinterpret_cast<const char*>(a.st_e) + wsrc,
                            wbytes, &full[s]);
        if (AP) tma_load_1d(dst + a.x_region + slot * a.w_region,
                            reinterpret_cast<const char*>(a.Vr[B.mode] + c0 * B.r), wbytes, &full[s]);
        if (hb == B.P)   // whole fibers: the group's columns are one contiguous range
          tma_load_1d(dst, xb + (B.off + c0 * B.P) * (i64)sizeof(T), xbytes, &full[s]);
      }
      if (hb != B.P) {
        __syncwarp();
        const unsigned seg = (unsigned)(hb * (i64)sizeof(T));
        for (i64 j = lane; j < nc; j += 32)
          tma_load_1d(dst + j * B.H * (i64)sizeof(T), xb + (B.off + (c0 + j) * B.P + r0) * (i64)sizeof(T), seg,
                      &full[s]);
      }
      __syncwarp();
      if (++s == a.nst) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else {
    // ---------------- consumers
    const double zeta = a.zetap ? __ldg(a.zetap) : a.zeta;
    double as[V][R], ae[V][R], ar[V][R];
    int pos[V];
    // A pass: the thread's rows [row, row + V) accumulate over its columns of the
    // band; flushed to its (block, CTA, column offset) slot at the band's end
    double* ap_dst = nullptr;
    int ap_f = -1, ap_r = R;
    auto ap_flush = [&]() {
      if (!AP || ap_dst == nullptr) return;
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (EX || q < ap_r) ap_dst[v * ap_r + q] = ar[v][q];
      ap_dst = nullptr;
    };
    double e2 = 0.0, x2 = 0.0, nfchk = 0.0;
    int cur_f = -1, cur_band = -1;
    int chunk = 0, coff = 0, H = 0, cpr = 1, mrows = 0, r = R;
    int s = 0;
    unsigned ph = 0;
    for (i64 t = t0; t < t1; ++t, advance()) {
      const FiberBlk& B = a.fb[cf];
      if (cf != cur_f) {
        if (SUMS && cur_f >= 0) {
          const double se = fb_cons_sum(e2, red, ncons), sx = fb_cons_sum(x2, red2, ncons);
          if (tid == 0) {
            a.partial[((i64)blockIdx.x * a.nblk + a.fb[cur_f].b) * 2] = se;
            a.partial[((i64)blockIdx.x * a.nblk + a.fb[cur_f].b) * 2 + 1] = sx;
          }
          e2 = 0.0;
          x2 = 0.0;
        }
        cur_f = cf;
        cur_band = -1;
        chunk = tid % B.nchB;
        coff = tid / B.nchB;
        H = B.H;
        cpr = B.cpr;
        mrows = B.mrows;
        r = EX ? R : B.r;
      }
      const int r0 = (int)cband * H;
      const int hb = min(H, (int)B.P - r0);
      const i64 c0 = ccg * B.CB;
      const int nc = (int)min((i64)B.CB, B.Q - c0);
      const bool act = coff < cpr && chunk * V < hb;
      const int row = r0 + chunk * V;
      if ((int)cband != cur_band || cf != ap_f) {
        ap_flush();
      }
      if ((int)cband != cur_band) {
        cur_band = (int)cband;
        if (AP && act) {
          ap_f = cf;
          ap_r = r;
          ap_dst = a.apart + B.pbase + ((i64)(blockIdx.x - B.c0) * cpr + coff) * B.P * r + (i64)row * r;
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int q = 0; q < R; ++q) ar[v][q] = 0.0;
        }
        if (act) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int rr = row + v;
            // row map (intersection copy: I_k; core: I_1); padded rows past Pv are
            // computed (finite) but never stored
            const int arow = B.amap ? __ldg(B.amap + (rr < B.Pv ? rr : B.Pv - 1)) : rr;
            if (WM) pos[v] = rr < B.Pv ? rr : -1;
            const bool live = !SC || rr < r0 + hb;   // (SC: rows past the column read x = 0 with zero A rows)
#pragma unroll
            for (int q = 0; q < R; ++q) {
              const bool on = (EX || q < r) && live;
              as[v][q] = (HS && on) ? __ldg(a.st_s + B.a_off + arow + (i64)q * B.dA) : 0.0;
              ae[v][q] = (HE && on) ? __ldg(a.st_e + B.a_off + arow + (i64)q * B.dA) : 0.0;
            }
          }
        }
      }
      mbar_wait(&full[s], ph);
      if (act) {
        const unsigned char* sb = ring + s * stage_bytes;
        const T* xs = reinterpret_cast<const T*>(sb) + chunk * V;
        const double* wss = reinterpret_cast<const double*>(sb + a.x_region);
        const double* wes = reinterpret_cast<const double*>(sb + a.x_region + (HS ? a.w_region : 0));   // W_e or V
        double* Mc = WM ? a.M[B.mode] + (c0 + coff) * (i64)mrows : nullptr;
        const i64 mstep = (i64)cpr * mrows;
        constexpr int CU = FB_COL_UNROLL;
#pragma unroll CU
        for (int jj = coff; jj < nc; jj += cpr) {
          VT xv;
          if (SC) {
#pragma unroll
            for (int v = 0; v < V; ++v) xv.v[v] = chunk * V + v < hb ? xs[jj * H + v] : (T)0;
          } else {
            xv = *reinterpret_cast<const VT*>(xs + jj * H);
          }
          double ws[R], we[R];
          if (EX && R % 2 == 0) {   // exact even rank: the column's rows are 16-byte aligned
            const double2* ws2 = reinterpret_cast<const double2*>(wss + jj * R);
            const double2* we2 = reinterpret_cast<const double2*>(wes + jj * R);
#pragma unroll
            for (int q = 0; q < R / 2; ++q) {
              if (HS) {
                const double2 t = ws2[q];
                ws[2 * q] = t.x;
                ws[2 * q + 1] = t.y;
              } else {
                ws[2 * q] = ws[2 * q + 1] = 0.0;
              }
              if (HE || AP) {
                const double2 t = we2[q];
                we[2 * q] = t.x;
                we[2 * q + 1] = t.y;
              } else {
                we[2 * q] = we[2 * q + 1] = 0.0;
              }
            }
          } else {
#pragma unroll
            for (int q = 0; q < R; ++q) {
              ws[q] = (HS && (EX || q < r)) ? wss[jj * r + q] : 0.0;
              we[q] = ((HE || AP) && (EX || q < r)) ? wes[jj * r + q] : 0.0;
            }
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const double x = (double)xv.v[v];
            double ls = 0.0, le = 0.0;
#pragma unroll
            for (int q = 0; q < R; ++q) {
              if (EX || q < r) {
                if (HS) ls = fma(as[v][q], ws[q], ls);
                if (HE) le = fma(ae[v][q], we[q], le);
              }
            }
            const double sv = fabs(x - ls) <= zeta ? 0.0 : x - ls;
            if (WM) {
              const double c = x - sv;
              nfchk = fma(c, 0.0, nfchk);   // NaN once any value is not finite
              if (pos[v] >= 0) Mc[pos[v]] = c;
            }
            if (SUMS) {
              const double rr = x - le - sv;
              e2 = fma(rr, rr, e2);
              x2 = fma(x, x, x2);
            }
            if (AP) {
              const double c = x - sv;
#pragma unroll
              for (int q = 0; q < R; ++q)
                if (EX || q < r) ar[v][q] = fma(c, we[q], ar[v][q]);
            }
          }
          if (WM) Mc += mstep;
        }
      }
      __syncwarp();
      if (lane == 0) fb_arrive(&empty[s]);
      if (++s == a.nst) {
        s = 0;
        ph ^= 1u;
      }
    }
    ap_flush();
    bad = !(nfchk == 0.0);
    if (SUMS && cur_f >= 0) {
      const double se = fb_cons_sum(e2, red, ncons), sx = fb_cons_sum(x2, red2, ncons);
      if (tid == 0) {
        a.partial[((i64)blockIdx.x * a.nblk + a.fb[cur_f].b) * 2] = se;
        a.partial[((i64)blockIdx.x * a.nblk + a.fb[cur_f].b) * 2 + 1] = sx;
      }
    }
  }
  if (WM && bad) atomicExch(a.nonfinite, 1);
  if (!SUMS) return;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    am_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // per-block sums over the CTAs' partials, every (block, sum) at once: thread t adds
  // the partials of CTAs t, t + blockDim, ... (all loads in flight together), a fixed
  // shuffle tree per warp, then the warps in order -- the operation order of one
  // block_sum per value (deterministic), without its serial per-value round trips
  {
    constexpr int NVAL = 2 * RT_MAX_MODES;
    __shared__ double redf[NVAL][FB_MAX_CONS / 32 + 1];
    double acc[NVAL];
#pragma unroll
    for (int v = 0; v < NVAL; ++v) acc[v] = 0.0;
    for (int c = tid; c < (int)gridDim.x; c += blockDim.x) {
      const volatile double* pc = reinterpret_cast<const volatile double*>(a.partial) + (i64)c * a.nblk * 2;
#pragma unroll
      for (int f = 0; f < RT_MAX_MODES; ++f)
        if (f < a.nfb) {
          const int b = a.fb[f].b;
          acc[2 * f] += pc[2 * b];
          acc[2 * f + 1] += pc[2 * b + 1];
        }
    }
    const int wid = tid >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int v = 0; v < NVAL; ++v)
      if (v < 2 * a.nfb) {   // (block-uniform)
        const double s = warp_sum(acc[v]);
        if (lane == 0) redf[v][wid] = s;
      }
    __syncthreads();
    if (tid < 2 * a.nfb) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += redf[tid][w];
      a.sums[2 * a.fb[tid >> 1].b + (tid & 1)] = t;
    }
  }
  if (tid == 0) *a.counter = 0u;
}

// ------------------------------------------------------------------ host planning

inline bool fb_block_ok(const Geom& g, int b, int dtype) {
  const int E = dtype == 0 ? 8 : 4;
  const BlockDesc& bd = g.blk[b];
  if (bd.r > FB_MAX_R || (bd.off * E) % 16 != 0 || bd.Q <= 0) return false;
  if (bd.is_core) return bd.P <= FB_MAX_CONS;   // error pass only: one band of scalar rows
  return (bd.P * E) % 16 == 0;
}

// one handled block as the pass sees it (the fiber block, or its intersection copy)
struct FbIn {
  i64 off, P, Q, w_off, a_off, dA;
  const int* amap;
  int Pv, b, mode, r, mrows;
  bool sc;   // columns not 16-byte multiples: scalar rows
};

// A_k[p, q] = siginv_q * sum over the CTAs whose tiles cover p's band (and their
// column offsets) of the A-pass partial rows: a warp per output, lanes over the
// terms, fixed-order shuffle tree (deterministic).
static __global__ void __launch_bounds__(256) k_fiber_areduce(FiberArgs a, int G) {
  if (rt_stopped(a.stop)) return;
  const int f = blockIdx.y;
  if (f >= a.nfb) return;
  const FiberBlk& B = a.fb[f];
  // a warp takes 8 consecutive outputs x 4 slices of the terms: lanes 8 s + j read output
  // o0 + j of slot s, s + 4, ... -- 64 contiguous bytes per slot (whole sectors), four
  // partial sums per output combined by a fixed two-step shuffle tree (deterministic)
  const int r = B.r, lane = threadIdx.x & 31, oj = lane & 7, sl = lane >> 3;
  const i64 nout = B.P * r;
  const i64 wstride = (i64)gridDim.x * (blockDim.x >> 5) * 8;
  for (i64 o0 = (blockIdx.x * (i64)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 8; o0 < nout; o0 += wstride) {
    const i64 o = o0 + oj;
    const bool on = o < nout;
    const i64 p = on ? o / r : 0;
    const int q = on ? (int)(o - p * r) : 0;
    double sum = 0.0;
    if (on) {
      const i64 t_lo = B.tfirst + (p / B.H) * B.ncg, t_hi = t_lo + B.ncg - 1;
      const i64 c_lo = ap_cta_of(t_lo, a.ntiles, G), c_hi = ap_cta_of(t_hi, a.ntiles, G);
      const i64 nterm = (c_hi - c_lo + 1) * B.cpr;
      const double* base = a.apart + B.pbase + (c_lo - B.c0) * B.cpr * B.P * r + o;
      for (i64 k = sl; k < nterm; k += 4) sum += base[k * B.P * r];   // slot (c, offset) = c_lo * cpr + k
    }
    sum += __shfl_xor_sync(0xffffffffu, sum, 8);
    sum += __shfl_xor_sync(0xffffffffu, sum, 16);
    if (on && sl == 0) a.a_out[B.a_off + p + (i64)q * B.dA] = sum * a.siginv[B.mode][q];
  }
}

template <typename T, int R, bool EX, bool HS, bool HE, bool AP, bool SC>
static int fb_launch_one(FiberArgs& fa, const FbIn* in, int nin, i64 apart_cap, cudaStream_t st) {
  constexpr int NS = (HS ? 1 : 0) + ((HE || AP) ? 1 : 0);
  constexpr int V = SC ? fb_sc_vec(R, fb_nsreg<HS, HE, AP>()) : fb_vec<T>(R, fb_nsreg<HS, HE, AP>());
  const int E = (int)sizeof(T);
  const int VA = SC ? 1 : 16 / E;   // bulk-copy segments are 16-byte multiples (SC: one band)
  // per-block bands / thread mapping
  int maxch = 1;
  i64 H[RT_MAX_MODES];
  int nch[RT_MAX_MODES];
  for (int f = 0; f < nin; ++f) {
    const i64 Pb = in[f].P;
    const i64 hmax = (i64)FB_MAX_CONS * V;
    const i64 nbands = (Pb + hmax - 1) / hmax;
    H[f] = ((Pb + nbands - 1) / nbands + VA - 1) / VA * VA;
    nch[f] = (int)((H[f] + V - 1) / V);
    maxch = std::max(maxch, nch[f]);
  }
  const int ncons = maxch > FB_MAX_CONS / 2 ? (maxch + 31) / 32 * 32 : FB_MAX_CONS;
  fa.nfb = nin;
  i64 t = 0, xreg = 16, wreg = 16;
  for (int f = 0; f < nin; ++f) {
    const FbIn& I = in[f];
    FiberBlk& B = fa.fb[f];
    B.off = I.off;
    B.P = I.P;
    B.Q = I.Q;
    B.dA = I.dA;
    B.amap = I.amap;
    B.Pv = I.Pv;
    B.w_off = I.w_off;
    B.a_off = I.a_off;
    B.H = (int)H[f];
    B.nchB = nch[f];
    B.cpr = std::max(1, ncons / nch[f]);
    i64 unit = B.cpr % 2 ? 2 * B.cpr : B.cpr;   // multiple of cpr, even (16-byte aligned W rows)
    if (SC) {   // and every tile's x start 16-byte aligned
      const i64 cb = I.P * E;
      i64 gcd = 16, x = cb % 16;
      while (x) { const i64 t2 = gcd % x; gcd = x; x = t2; }
      const i64 au = 16 / gcd;
      i64 a = unit, b2 = au;
      while (b2) { const i64 t2 = a % b2; a = b2; b2 = t2; }
      unit = unit / a * au;
    }
    const i64 colb = H[f] * E + (i64)NS * I.r * 8;
    static const i64 stage_bytes = [] {
      const char* v = getenv("RTCUR_FB_STAGE_KB");
      return v ? std::max<i64>(1, atoll(v)) * 1024 : (i64)FB_STAGE_BYTES;
    }();
    i64 CB = std::max<i64>(1, stage_bytes / colb) / unit * unit;
    if (CB == 0) CB = unit;
    B.CB = (int)CB;
    const i64 nbands = (I.P + H[f] - 1) / H[f];
    B.ncg = (I.Q + CB - 1) / CB;
    B.nbands = (int)nbands;
    B.tfirst = t;
    t += nbands * B.ncg;
    B.b = I.b;
    B.mode = I.mode;
    B.r = I.r;
    B.mrows = I.mrows;
    xreg = std::max<i64>(xreg, (CB * H[f] * E + 15) & ~15LL);
    wreg = std::max<i64>(wreg, (CB * I.r * 8 + 15) & ~15LL);
  }
  fa.ntiles = t;
  fa.x_region = (int)((xreg + 127) & ~127LL);
  fa.w_region = (int)((wreg + 127) & ~127LL);
  const i64 stage = fa.x_region + (i64)NS * fa.w_region;
  // shared-memory ring per CTA: the budget decides how many CTAs share an SM
  // (RTCUR_FB_SMEM_KB overrides; default two CTAs per SM)
  i64 budget = FB_SMEM_BUDGET;
  if (const char* env = getenv("RTCUR_FB_SMEM_KB")) budget = std::max<i64>(16, atoll(env)) * 1024;
  fa.nst = (int)std::min<i64>(FB_MAX_STAGES, budget / stage);
  if (fa.nst < 2) fa.nst = 2;
  const int smem = 2 * FB_MAX_STAGES * 8 + (int)(fa.nst * stage);
  if (smem > 227 * 1024) return -(int)cudaErrorInvalidConfiguration;
  auto K = k_fiber_pass<T, R, EX, HS, HE, AP, SC>;
  cudaError_t e = raise_dyn_smem_once<k_fiber_pass<T, R, EX, HS, HE, AP, SC>>();
  if (e != cudaSuccess) return -(int)e;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K, ncons + 32, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  per_sm = std::min(per_sm, FB_MAX_CTAS_PER_SM);
  const int grid = (int)std::max<i64>(1, std::min<i64>((i64)std::max(1, 148 - fa.reserve_sms) * per_sm, t));
  i64 maxpr = 1;
  if (AP) {   // partial slots: one P x r slot per (block, CTA touching it)
    i64 pb = 0;
    for (int f = 0; f < nin; ++f) {
      FiberBlk& B = fa.fb[f];
      const i64 c0 = ap_cta_of(B.tfirst, t, grid), c1 = ap_cta_of(B.tfirst + (i64)B.nbands * B.ncg - 1, t, grid);
      B.c0 = (int)c0;
      B.pbase = pb;
      pb += (c1 - c0 + 1) * B.cpr * B.P * B.r;
      maxpr = std::max<i64>(maxpr, B.P * B.r);
    }
    if (pb > apart_cap) return -(int)cudaErrorInvalidValue;
  }
  K<<<grid, ncons + 32, smem, st>>>(fa);
  e = cudaGetLastError();
  if (e != cudaSuccess) return -(int)e;
  if (AP) {
    k_fiber_areduce<<<dim3((unsigned)std::min<i64>((maxpr + 63) / 64, 1024), nin), 256, 0, st>>>(fa, grid);
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? (AP ? 2 : 1) : -(int)e;   // kernels launched
}

template <typename T, int R, bool EX>
static int fb_launch_states(FiberArgs& fa, const FbIn* in, int nin, bool hs, bool he, bool ap, i64 cap,
                            cudaStream_t st) {
  if (in[0].sc) {   // scalar rows: the error pass over the core only
    if (!he || ap) return -(int)cudaErrorInvalidValue;
    return hs ? fb_launch_one<T, R, EX, true, true, false, true>(fa, in, nin, cap, st)
              : fb_launch_one<T, R, EX, false, true, false, true>(fa, in, nin, cap, st);
  }
  if (ap) return hs ? fb_launch_one<T, R, EX, true, false, true, false>(fa, in, nin, cap, st)
                    : fb_launch_one<T, R, EX, false, false, true, false>(fa, in, nin, cap, st);
  if (hs && he) return fb_launch_one<T, R, EX, true, true, false, false>(fa, in, nin, cap, st);
  if (hs) return fb_launch_one<T, R, EX, true, false, false, false>(fa, in, nin, cap, st);
  if (he) return fb_launch_one<T, R, EX, false, true, false, false>(fa, in, nin, cap, st);
  return fb_launch_one<T, R, EX, false, false, false, false>(fa, in, nin, cap, st);
}

template <typename T>
static int fb_launch_t(const FiberLaunch& L, unsigned mask, cudaStream_t st) {
  FiberArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.stop = L.g.stop;
  fa.reserve_sms = L.reserve_sms;
  fa.st_s = L.st_s;
  fa.st_e = L.st_e;
  fa.zeta = L.zeta;
  fa.zetap = L.zetap;
  for (int m = 0; m < RT_MAX_MODES; ++m) {
    fa.M[m] = L.M[m];
    fa.rowpos[m] = L.rowpos[m];
  }
  fa.partial = L.partial;
  fa.sums = L.sums;
  fa.counter = L.counter;
  fa.nonfinite = L.nonfinite;
  const bool hs = L.st_s != nullptr, he = L.st_e != nullptr, ap = L.ap != 0;
  for (int m = 0; m < RT_MAX_MODES; ++m) {
    fa.Vr[m] = L.Vr[m];
    fa.siginv[m] = L.siginv[m];
  }
  fa.apart = L.apart;
  fa.a_out = L.a_out;
  // A pass and error pass: the whole fiber blocks; threshold pass: the intersection copies X(I_k, J_k) (only those rows feed M_k);
  // error pass: the whole fiber blocks
  FbIn in[RT_MAX_MODES];
  int nin = 0, rmax = 1, rmin = 64;
  fa.xb = (he || ap) ? L.xb : L.xi;
  fa.nblk = L.g.nblk;
  const int E = (int)sizeof(T);
  for (int b = he ? 0 : 1; b < L.g.nblk; ++b) {   // the core only in the error pass
    if (!(mask >> b & 1)) continue;
    const BlockDesc& bd = L.g.blk[b];
    const int m = bd.mode;
    FbIn& I = in[nin++];
    I.sc = (bd.P * E) % 16 != 0;
    I.Q = bd.Q;
    I.w_off = bd.w_off;
    I.a_off = L.g.a_off[m];
    I.dA = L.g.dim[m];
    I.b = b;
    I.mode = m;
    I.r = bd.r;
    I.mrows = (int)L.g.nrows[m];
    if (he || ap) {
      I.off = bd.off;
      I.P = bd.P;
      I.Pv = (int)bd.P;
      I.amap = bd.is_core ? L.rows[0] : nullptr;   // core rows are I_1
    } else {
      I.off = L.xi_off[m];
      I.P = L.xi_ld[m];
      I.Pv = (int)L.g.nrows[m];
      I.amap = L.rows[m];
    }
    rmax = std::max(rmax, bd.r);
    rmin = std::min(rmin, bd.r);
  }
  (void)rmin;
  (void)rmax;
  // one launch per distinct rank (exact unrolled dot products; buckets for the rest)
  bool done[RT_MAX_MODES] = {};
  int nl = 0;
  for (int f = 0; f < nin; ++f) {
    if (done[f]) continue;
    FbIn grp[RT_MAX_MODES];
    int ng = 0;
    const int rk = in[f].r;
    const bool sc = in[f].sc;
    for (int h = f; h < nin; ++h)
      if (!done[h] && in[h].r == rk && in[h].sc == sc) {
        grp[ng++] = in[h];
        done[h] = true;
      }
    FiberArgs fg = fa;
    int st_ = 0;
    switch (rk) {
#define FB_EXACT(k)                                                                           \
  case k:                                                                                     \
    st_ = fb_launch_states<T, k, true>(fg, grp, ng, hs, he, ap, L.apart_cap, st);             \
    break;
      FB_EXACT(1) FB_EXACT(2) FB_EXACT(3) FB_EXACT(4) FB_EXACT(5) FB_EXACT(6) FB_EXACT(8) FB_EXACT(10)
      FB_EXACT(16)
#undef FB_EXACT
      default:
        st_ = rk <= 8 ? fb_launch_states<T, 8, false>(fg, grp, ng, hs, he, ap, L.apart_cap, st)
                      : fb_launch_states<T, 16, false>(fg, grp, ng, hs, he, ap, L.apart_cap, st);
        break;
    }
    if (st_ < 0) return st_;
    nl += st_;
  }
  return nl;
}

// Intersection copies for the threshold pass: xi_k[i + q * ld_k] = x_k(I_k[i], q)
// from the compact fiber block (rows past |I_k| zero).  One CTA row per (mode, column chunk).
template <typename T>
__global__ void __launch_bounds__(256) k_xi_extract(FiberLaunch L, unsigned mask) {
  if (rt_stopped(L.g.stop)) return;
  const int b = blockIdx.y + 1;
  if (b >= L.g.nblk || !(mask >> b & 1)) return;
  const BlockDesc& bd = L.g.blk[b];
  const int m = bd.mode;
  const i64 ld = L.xi_ld[m], nr = L.g.nrows[m];
  const T* src = reinterpret_cast<const T*>(L.xb) + bd.off;
  T* dst = reinterpret_cast<T*>(const_cast<void*>(L.xi)) + L.xi_off[m];
  const int* rows = L.rows[m];
  const i64 n = ld * bd.Q;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
    const i64 q = e / ld, i = e - q * ld;
    dst[e] = i < nr ? src[(i64)__ldg(rows + i) + q * bd.P] : (T)0;
  }
}

template <typename T>
static int fb_extract_t(const FiberLaunch& L, unsigned mask, cudaStream_t st) {
  i64 mx = 1;
  for (int b = 1; b < L.g.nblk; ++b)
    if (mask >> b & 1) mx = std::max<i64>(mx, L.xi_ld[L.g.blk[b].mode] * L.g.blk[b].Q);
  dim3 grid((unsigned)std::min<i64>((mx + 255) / 256, 592), L.g.nblk - 1);
  k_xi_extract<T><<<grid, 256, 0, st>>>(L, mask);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}
