// k_full_tma.cu -- K3 with the X stream staged by TMA bulk copies.
//
// Same result as k_full (k_full.cu) -- the reference's full-output step
//   L = cur_reconstruct_full(cur)           (cli.py:238 -> fiber_cur.py:277-285)
//   S = hard_threshold(x - L, zeta_final)    (cli.py:240-242)
// with the residual sums, bit-identical per element (same FMA order) -- but
// mapped so the per-element work is r_1 register FMAs:
//
//  * a CTA owns a band of mode-1 rows [b*H, b*H+H) and a contiguous range of
//    column groups (CB mode-1 fibers each); each consumer thread owns V
//    consecutive rows (one 16-byte vector) and keeps their A_1 rows in
//    registers (V*r_1 doubles) for the whole band;
//  * a producer warp streams the band's fiber segments of X into an
//    NST-deep shared-memory ring with cp.async.bulk (one copy per column
//    group when the band is the whole fiber, since the columns are then
//    contiguous in memory), full/empty mbarriers per slot;
//  * per fiber, the r_1 values of Tf are warp-uniform L1 loads, and L and S
//    go straight from registers to HBM as 16-byte coalesced stores.
//
// HBM traffic is the algorithmic 3*E*N (read X, write L and S); nothing is
// re-read.  Envelope: (hi-lo)*E % 16 == 0, 16-byte aligned X/L/S, r_1 <= 16.
#include <algorithm>
#include <cstdlib>
#include "bp_types.cuh"
#include "full_types.cuh"

#define FT_MAX_CONSUMERS 384
#define FT_STAGE_BYTES (32 * 1024)
#define FT_SMEM_BUDGET (200 * 1024)
#define FT_MAX_STAGES 8

struct FullTmaArgs {
  const void* X;
  void* L;
  void* S;
  const double* A1;     // A_1 + lo (rows of this slab), column-major with leading dimension d1
  const double* Tf;     // ncols x r1 row-major
  i64 d1;
  i64 ld;               // rows of the slab
  i64 ncols;
  i64 ntiles, ncg;      // tiles = bands x column groups (column group fastest)
  int H, nchB, cpr, CB, nst;
  double zeta;
  double* partial;
  double* sums;
  unsigned int* counter;
};

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// V consecutive elements moved as one aligned vector (16 or 8 bytes)
template <typename T, int V>
struct alignas(V * sizeof(T)) VecN {
  T v[V];
};

template <typename T, int R, int V>
__global__ void __launch_bounds__(FT_MAX_CONSUMERS + 32, 1) k_full_tma(FullTmaArgs a) {
  typedef VecN<T, V> VT;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ double red[(FT_MAX_CONSUMERS + 32) / 32];
  __shared__ bool am_last;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm);
  unsigned long long* empty = full + FT_MAX_STAGES;
  unsigned char* ring = sm + 2 * FT_MAX_STAGES * 8;
  const int tid = threadIdx.x;
  const int ncons = blockDim.x - 32;
  const int lane = tid & 31;
  const i64 x_bytes = (i64)a.CB * a.H * (i64)sizeof(T);
  const i64 stage_bytes = x_bytes + (((i64)a.CB * R * 8 + 15) & ~15LL);
  const bool has_x = a.X != nullptr;
  if (tid == 0) {
    for (int s = 0; s < a.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const i64 t0 = a.ntiles * blockIdx.x / gridDim.x, t1 = a.ntiles * (blockIdx.x + 1) / gridDim.x;
  double e2 = 0.0, x2 = 0.0;
  if (tid >= ncons) {
    // ---------------- producer warp: stream the tiles' X segments and Tf rows into the ring
    {
      const char* X = reinterpret_cast<const char*>(a.X);
      for (i64 t = t0, k = 0; t < t1; ++t, ++k) {
        const int s = (int)(k % a.nst);
        if (k >= a.nst) mbar_wait(&empty[s], (unsigned)((k / a.nst - 1) & 1));
        const i64 band = t / a.ncg, cg = t - band * a.ncg;
        const i64 r0 = band * a.H;
        const i64 hb = min((i64)a.H, a.ld - r0);
        const i64 c0 = cg * a.CB;
        const i64 nc = min((i64)a.CB, a.ncols - c0);
        unsigned char* dst = ring + s * stage_bytes;
        // Tf rows of the group: contiguous, 16-byte aligned (CB even), size rounded up
        // to 16 bytes (the Tf scratch is padded, rtcur_engine_full_scratch_bytes)
        const unsigned tf_bytes = (unsigned)((nc * R * 8 + 15) & ~15LL);
        if (!has_x) {
          if (lane == 0) {
            mbar_expect_tx(&full[s], tf_bytes);
            tma_load_1d(dst + x_bytes, a.Tf + c0 * R, tf_bytes, &full[s]);
          }
        } else if (hb == a.ld) {   // whole fibers: the column group is one contiguous range
          if (lane == 0) {
            const unsigned bytes = (unsigned)(nc * a.ld * (i64)sizeof(T));
            mbar_expect_tx(&full[s], bytes + tf_bytes);
            tma_load_1d(dst, X + c0 * a.ld * (i64)sizeof(T), bytes, &full[s]);
            tma_load_1d(dst + x_bytes, a.Tf + c0 * R, tf_bytes, &full[s]);
          }
        } else {
          const unsigned seg = (unsigned)(hb * (i64)sizeof(T));
          if (lane == 0) {
            mbar_expect_tx(&full[s], seg * (unsigned)nc + tf_bytes);
            tma_load_1d(dst + x_bytes, a.Tf + c0 * R, tf_bytes, &full[s]);
          }
          __syncwarp();
          for (i64 j = lane; j < nc; j += 32)
            tma_load_1d(dst + j * a.H * (i64)sizeof(T), X + ((c0 + j) * a.ld + r0) * (i64)sizeof(T), seg, &full[s]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- consumers: V rows x (every cpr-th fiber of the group) per thread
    const int chunk = tid % a.nchB, coff = tid / a.nchB;
    const bool in_map = coff < a.cpr;
    const double zeta = a.zeta;
    T* Lp = reinterpret_cast<T*>(a.L);
    T* Sp = reinterpret_cast<T*>(a.S);
    double A[V][R];
    i64 cur_band = -1;
    for (i64 t = t0, k = 0; t < t1; ++t, ++k) {
      const int s = (int)(k % a.nst);
      const i64 band = t / a.ncg, cg = t - band * a.ncg;
      const i64 r0 = band * a.H;
      const i64 hb = min((i64)a.H, a.ld - r0);
      const i64 c0 = cg * a.CB;
      const i64 nc = min((i64)a.CB, a.ncols - c0);
      const bool act = in_map && (i64)chunk * V < hb;
      const i64 row = r0 + (i64)chunk * V;
      if (band != cur_band) {
        cur_band = band;
        if (act) {
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int q = 0; q < R; ++q) A[v][q] = __ldg(a.A1 + row + v + (i64)q * a.d1);
        }
      }
      mbar_wait(&full[s], (unsigned)((k / a.nst) & 1));
      if (act) {
        const unsigned char* src = ring + s * stage_bytes + ((i64)chunk * V) * (i64)sizeof(T);
        const double* tfs = reinterpret_cast<const double*>(ring + s * stage_bytes + x_bytes);
        for (i64 jj = coff; jj < nc; jj += a.cpr) {
          const i64 col = c0 + jj;
          VT xv;
          if (has_x) xv = *reinterpret_cast<const VT*>(src + jj * a.H * (i64)sizeof(T));
          double tf[R];
#pragma unroll
          for (int q = 0; q < R; ++q) tf[q] = tfs[jj * R + q];
          VT lv, sv;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            double l = 0.0;
#pragma unroll
            for (int q = 0; q < R; ++q) l = fma(A[v][q], tf[q], l);
            const double x = has_x ? (double)xv.v[v] : 0.0;
            const double sp = hard_thr(x - l, zeta);
            const double res = x - l - sp;
            e2 = fma(res, res, e2);
            x2 = fma(x, x, x2);
            lv.v[v] = (T)l;
            sv.v[v] = (T)sp;
          }
          const i64 e = col * a.ld + row;
          if (Lp) *reinterpret_cast<VT*>(Lp + e) = lv;
          if (Sp) *reinterpret_cast<VT*>(Sp + e) = sv;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  e2 = block_sum(e2, red);
  x2 = block_sum(x2, red);
  if (tid == 0) {
    a.partial[2 * blockIdx.x] = e2;
    a.partial[2 * blockIdx.x + 1] = x2;
    __threadfence();
    am_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double se = 0.0, sx = 0.0;
  for (int c = tid; c < (int)gridDim.x; c += blockDim.x) {
    se += ((volatile double*)a.partial)[2 * c];
    sx += ((volatile double*)a.partial)[2 * c + 1];
  }
  se = block_sum(se, red);
  sx = block_sum(sx, red);
  if (tid == 0) {
    a.sums[0] = se;
    a.sums[1] = sx;
    *a.counter = 0u;
  }
}

template <typename T, int R, int V>
static int launch_one(const FullTmaArgs& ta, int grid, int threads, int smem, cudaStream_t st) {
  auto F = k_full_tma<T, R, V>;
  cudaError_t e = raise_dyn_smem_once<k_full_tma<T, R, V>>();
  if (e != cudaSuccess) return -(int)e;
  F<<<grid, threads, smem, st>>>(ta);
  e = cudaGetLastError();
  return e == cudaSuccess ? 1 : -(int)e;
}

// elements per thread: 16-byte vectors while V*R <= 32 doubles of A rows fit the
// register budget, else 8-byte vectors
template <typename T>
__host__ __device__ constexpr int ft_vec(int r) {
  return (int)(16 / sizeof(T)) * r <= 32 ? (int)(16 / sizeof(T)) : (int)(8 / sizeof(T));
}

template <typename T>
static int launch_r(int r, const FullTmaArgs& ta, int grid, int threads, int smem, cudaStream_t st) {
  switch (r) {
#define FT_CASE(k) \
  case k:          \
    return launch_one<T, k, ft_vec<T>(k)>(ta, grid, threads, smem, st);
    FT_CASE(1) FT_CASE(2) FT_CASE(3) FT_CASE(4) FT_CASE(5) FT_CASE(6) FT_CASE(7) FT_CASE(8)
    FT_CASE(9) FT_CASE(10) FT_CASE(11) FT_CASE(12) FT_CASE(13) FT_CASE(14) FT_CASE(15) FT_CASE(16)
#undef FT_CASE
    default:
      return 0;
  }
}

int full_tma_launch(const FullArgs& a, int max_grid, cudaStream_t st) {
  const int E = a.dtype == 0 ? 8 : 4;
  const int V = a.dtype == 0 ? ft_vec<double>(a.r1) : ft_vec<float>(a.r1);
  const int VA = 16 / E;   // TMA segments are 16-byte multiples
  const i64 ld = a.hi - a.lo;
  if (const char* env = getenv("RTCUR_K3_GENERIC")) {
    if (env[0] == '1') return 0;
  }
  if (a.r1 < 1 || a.r1 > 16 || ld <= 0 || a.ncols <= 0 || (ld * E) % 16 != 0) return 0;
  auto aligned = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  if (!aligned(a.X) || !aligned(a.L) || !aligned(a.S)) return 0;
  const i64 hmax = (i64)FT_MAX_CONSUMERS * V;
  const i64 nb = (ld + hmax - 1) / hmax;
  const i64 H = ((ld + nb - 1) / nb + VA - 1) / VA * VA;
  const int nchB = (int)(H / V);
  const int cpr = std::max(1, FT_MAX_CONSUMERS / nchB);   // fibers in flight per thread row
  const int ncons = (cpr * nchB + 31) / 32 * 32;
  const i64 col_bytes = H * E + a.r1 * 8;
  const i64 unit = cpr % 2 ? 2 * cpr : cpr;   // CB: a multiple of cpr, even (aligned Tf rows)
  i64 CB = std::max<i64>(1, FT_STAGE_BYTES / col_bytes) / unit * unit;
  if (CB == 0) CB = unit;
  const i64 stage = CB * H * E + ((CB * a.r1 * 8 + 15) & ~15LL);
  int nst = (int)std::min<i64>(FT_MAX_STAGES, FT_SMEM_BUDGET / stage);
  if (nst < 2) return 0;
  const i64 ncg = (a.ncols + CB - 1) / CB;
  const i64 ntiles = nb * ncg;
  int grid = (int)std::min<i64>(std::min<i64>(148, max_grid), ntiles);
  const int smem = 2 * FT_MAX_STAGES * 8 + (int)(nst * stage);
  FullTmaArgs ta;
  ta.X = a.X;
  ta.L = a.L;
  ta.S = a.S;
  ta.A1 = a.A1 + a.lo;
  ta.Tf = a.Tf;
  ta.d1 = a.d1;
  ta.ld = ld;
  ta.ncols = a.ncols;
  ta.ntiles = ntiles;
  ta.ncg = ncg;
  ta.H = (int)H;
  ta.nchB = nchB;
  ta.cpr = cpr;
  ta.CB = (int)CB;
  ta.nst = nst;
  ta.zeta = a.zeta;
  ta.partial = a.partial;
  ta.sums = a.sums;
  ta.counter = a.counter;
  return a.dtype == 0 ? launch_r<double>(a.r1, ta, grid, ncons + 32, smem, st)
                      : launch_r<float>(a.r1, ta, grid, ncons + 32, smem, st);
}
