// k_core.cu -- the core block's passes for short columns (32 |I_1| E <= 11 KB):
//
//   G pass (mode 0):  t1[q, :] = sum_p U~_1[p, :] clean(p, q)            (fiber_cur.py:264-267
//                     via the Tucker collapse: the first contraction of G = clean_core x_i U~_i^T)
//   error pass (1):   sum (x - L_e - S)^2, sum x^2 over the core block      (solver.py:209-231)
//
// with, per entry (p, q) of the |I_1| x Q core (reference solver.py:336-355):
//   L_s = A_1^s[I_1(p), :] . W^s[q, :]   (previous iterate, the same fma order as eval_low)
//   S   = HT(x - L_s, zeta)              strict |.| > zeta keep (py_kernels.py:226-230)
//   clean = x - S,  L_e = A_1^e[I_1(p), :] . W^e[q, :]
//
// Layout.  The core is column-major with short columns (|I_1| entries), so a
// warp takes 32 whole columns at a time -- one contiguous run of 32 |I_1|
// elements -- copies it global -> shared with 16-byte cp.async (coalesced; one
// run per warp, 24 warps per SM at |I_1| = 65 fp32 hide each other's loads)
// and each lane then walks its own column down the rows: the
// column's W rows stay in registers, the |I_1| x r A (and U~) rows sit in
// shared memory and are read as warp broadcasts, and the column stride in
// shared memory (|I_1| elements, odd for the BASELINE shapes) keeps the
// lanes' reads conflict-free.  The G pass then owns each output row t1[q, :]
// outright (no cross-lane reduction); the error pass reduces per-CTA partials
// in CTA order (deterministic).  Algorithmic bytes per launch: E * |I_1| * Q
// of x plus the W rows (8 r Q per state).
#include <algorithm>

#include "bp_types.cuh"
#include "core_types.cuh"

#define CP_MAX_WARPS 8
#define CP_SMEM_BUDGET (200 * 1024)

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// bytes of shared memory ahead of the x buffers (A / U rows, reduction scratch)
__host__ __device__ inline size_t cp_fixed_bytes(int P, int R) {
  return (((size_t)2 * P * R + 2 * CP_MAX_WARPS) * 8 + 15) & ~(size_t)15;
}

template <typename T, int R, bool HS, int MODE>
__global__ void __launch_bounds__(CP_MAX_WARPS * 32, 3) k_core_pass(CoreLaunch c) {
  if (rt_stopped(c.stop)) return;
  extern __shared__ __align__(16) unsigned char csm[];
  const int P = c.P, r = c.r;
  double* As = reinterpret_cast<double*>(csm);   // P x R: A_1^s rows (threshold state)
  double* Bs = As + P * R;                        // P x R: A_1^e rows (error) or U~_1 rows (G pass)
  double* red = Bs + P * R;                       // 2 x CP_MAX_WARPS
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int xelems = 32 * P;                      // one run of 32 columns
  const int nbuf = c.nbuf;
  T* xb0 = reinterpret_cast<T*>(csm + cp_fixed_bytes(P, R)) + (size_t)wid * nbuf * xelems;
  T* xb1 = xb0 + (nbuf == 2 ? xelems : 0);
  for (int i = tid; i < P * r; i += blockDim.x) {
    const int p = i / r, a = i - p * r;
    const i64 row = c.rows0[p];
    if (HS) As[p * R + a] = c.st_s[c.a_off + row + a * c.dA];
    Bs[p * R + a] = MODE == 1 ? c.st_e[c.a_off + row + a * c.dA] : c.U[p * r + a];
  }
  __syncthreads();
  const double zeta = c.zetap ? *c.zetap : c.zeta;
  const i64 Q = c.Q;
  const i64 ngroups = (Q + 31) >> 5;
  const i64 gstride = (i64)gridDim.x * nw;
  const char* xg = reinterpret_cast<const char*>(c.x);
  const i64 run_bytes = (i64)xelems * (i64)sizeof(T);
  auto issue = [&](i64 g, T* buf) {
    const i64 n = min((i64)32, Q - 32 * g);
    const int chunks = (int)((n * P * (i64)sizeof(T) + 15) >> 4);
    const char* src = xg + g * run_bytes;
    char* dst = reinterpret_cast<char*>(buf);
    for (int i = lane; i < chunks; i += 32) cp_async16(dst + 16 * i, src + 16 * i);
  };
  double e2 = 0.0, x2 = 0.0;
  i64 g = (i64)blockIdx.x * nw + wid;
  if (nbuf == 2) {
    if (g < ngroups) issue(g, xb0);
    cp_commit();
  }
  for (int it = 0; g < ngroups; g += gstride, ++it) {
    T* cur = (it & 1) ? xb1 : xb0;
    if (nbuf == 2) {   // the next run streams in while this one is computed
      if (g + gstride < ngroups) issue(g + gstride, (it & 1) ? xb0 : xb1);
      cp_commit();
      cp_wait<1>();
    } else {           // single buffer: the other resident warps hide the load
      issue(g, xb0);
      cp_commit();
      cp_wait<0>();
    }
    __syncwarp();
    const i64 q = 32 * g + lane;
    if (q < Q) {
      double ws[R], wb[R], acc[R];
#pragma unroll
      for (int a = 0; a < R; ++a) {
        ws[a] = (HS && a < r) ? c.st_s[c.w_off + q * r + a] : 0.0;
        wb[a] = (MODE == 1 && a < r) ? c.st_e[c.w_off + q * r + a] : 0.0;
        acc[a] = 0.0;
      }
      const T* xc = cur + lane * P;
#pragma unroll 4
      for (int p = 0; p < P; ++p) {
        const double x = (double)xc[p];
        double ls = 0.0;
        if (HS) {
#pragma unroll
          for (int a = 0; a < R; ++a)
            if (a < r) ls = fma(As[p * R + a], ws[a], ls);
        }
        const double sv = fabs(x - ls) <= zeta ? 0.0 : x - ls;
        if (MODE == 0) {
          const double cl = x - sv;
#pragma unroll
          for (int a = 0; a < R; ++a)
            if (a < r) acc[a] = fma(Bs[p * R + a], cl, acc[a]);
        } else {
          double le = 0.0;
#pragma unroll
          for (int a = 0; a < R; ++a)
            if (a < r) le = fma(Bs[p * R + a], wb[a], le);
          const double rr = x - le - sv;
          e2 = fma(rr, rr, e2);
          x2 = fma(x, x, x2);
        }
      }
      if (MODE == 0) {
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (a < r) c.t1[q * r + a] = acc[a];
      }
    }
    __syncwarp();   // this buffer is refilled for the group after next
  }
  cp_wait<0>();
  if (MODE == 0) return;
  // error pass: CTA partials, then the last CTA sums them in CTA order (deterministic)
  e2 = warp_sum(e2);
  x2 = warp_sum(x2);
  if (lane == 0) {
    red[wid] = e2;
    red[CP_MAX_WARPS + wid] = x2;
  }
  __syncthreads();
  __shared__ bool am_last;
  if (tid == 0) {
    double se = 0.0, sx = 0.0;
    for (int w = 0; w < nw; ++w) {
      se += red[w];
      sx += red[CP_MAX_WARPS + w];
    }
    c.partial[2 * blockIdx.x] = se;
    c.partial[2 * blockIdx.x + 1] = sx;
    __threadfence();
    am_last = atomicAdd(c.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double se = 0.0, sx = 0.0;
  for (int b = tid; b < (int)gridDim.x; b += blockDim.x) {
    se += ((volatile double*)c.partial)[2 * b];
    sx += ((volatile double*)c.partial)[2 * b + 1];
  }
  se = block_sum(se, red);
  sx = block_sum(sx, red);
  if (tid == 0) {
    c.sums[0] = se;
    c.sums[1] = sx;
    *c.counter = 0u;
  }
}

bool core_pass_fits(int P, int r, int dtype) {
  const size_t esz = dtype == 0 ? 8 : 4;
  // lanes over columns needs many resident warps (the per-lane chains are
  // latency bound): a 32-column run must stay small enough for >= 16 warps per
  // SM (measured: 8 warps per SM is no faster than the block pass), r_1 <= 8
  return P >= 1 && r >= 1 && r <= 8 && (size_t)32 * P * esz <= 11 * 1024;
}

template <typename T, int R, bool HS, int MODE>
static int cp_launch_t(const CoreLaunch& c, cudaStream_t st) {
  auto kern = k_core_pass<T, R, HS, MODE>;
  // 8-warp CTAs, single-buffered runs (three CTAs per SM at |I_1| = 65 fp32)
  CoreLaunch cc = c;
  cc.nbuf = 1;
  const size_t per_warp = (size_t)32 * c.P * sizeof(T);
  const size_t fixed = cp_fixed_bytes(c.P, R);
  const int warps = CP_MAX_WARPS;
  const size_t smem = fixed + (size_t)warps * per_warp;
  cudaError_t e = raise_dyn_smem_once<k_core_pass<T, R, HS, MODE>>();
  if (e != cudaSuccess) return -(int)e;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const i64 ngroups = (c.Q + 31) / 32;
  const i64 grid = std::max<i64>(1, std::min<i64>((i64)148 * per_sm, (ngroups + warps - 1) / warps));
  kern<<<(unsigned)grid, warps * 32, smem, st>>>(cc);
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

template <typename T, int R>
static int cp_launch_r(const CoreLaunch& c, cudaStream_t st) {
  const bool hs = c.st_s != nullptr;
  if (c.mode == 0) return hs ? cp_launch_t<T, R, true, 0>(c, st) : cp_launch_t<T, R, false, 0>(c, st);
  return hs ? cp_launch_t<T, R, true, 1>(c, st) : cp_launch_t<T, R, false, 1>(c, st);
}

template <typename T>
static int cp_launch_d(const CoreLaunch& c, cudaStream_t st) {
  if (c.r <= 4) return cp_launch_r<T, 4>(c, st);
  return cp_launch_r<T, 8>(c, st);
}

int core_pass_launch(const CoreLaunch& c, cudaStream_t st) {
  if (!core_pass_fits(c.P, c.r, c.dtype)) return -(int)cudaErrorInvalidValue;
  return c.dtype == 0 ? cp_launch_d<double>(c, st) : cp_launch_d<float>(c, st);
}
