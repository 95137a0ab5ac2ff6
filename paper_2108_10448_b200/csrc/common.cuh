// common.cuh -- shared definitions for the RTCUR sm_100a kernels.
//
// Layout contract (reference tensor.py:1-10): the observed tensor is a flat
// buffer with mode 1 varying fastest.  All index sets on the device are
// 0-based (the host converts the reference's 1-based sets once per draw).
// Every low-rank quantity (G, A_k, W_b, SVD factors) is float64 regardless of
// the storage dtype of X, so fp32 tensors are processed with fp64 arithmetic
// (the reference is fp64-only, tensor.py:8).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

// Raise a kernel's dynamic shared-memory limit to the device's opt-in maximum
// (minus its static shared memory), once per kernel and device (function
// attributes are per device context).  Per-launch cudaFuncSetAttribute calls
// with the launch's own size race between host threads launching the same
// kernel with different sizes (a second thread can lower the limit between the
// first thread's set and launch: "invalid argument").
#define RT_MAX_DEVICES 64
template <auto Kernel>   // one table per kernel (not per signature)
inline cudaError_t raise_dyn_smem_once() {
  static std::atomic<int> state[RT_MAX_DEVICES];   // 0 unset, 1 + cudaError_t once done
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= RT_MAX_DEVICES) return cudaErrorInvalidDevice;
  const int st = state[dev].load(std::memory_order_acquire);
  if (st) return (cudaError_t)(st - 1);
  int optin = 227 * 1024;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, Kernel);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  state[dev].store(1 + (int)e, std::memory_order_release);   // idempotent: racing setters write the same limit
  return e;
}

#define RT_MAX_MODES 8
#define RT_MAX_BLOCKS (RT_MAX_MODES + 1)
#define RT_MAX_RANK 32
#define RT_EIG_MAX_N 237   // packed lower triangle of 237x237 fp64 fits 227 KB smem

// status codes (mapped to Python exceptions by the host layer)
#define RT_OK 0
#define RT_ERR_VALUE 1      // ValueError
#define RT_ERR_INDEX 2      // IndexError
#define RT_ERR_ARITH 3      // ArithmeticError
#define RT_ERR_CUDA 4       // RuntimeError (CUDA failure)
#define RT_ERR_UNSUPPORTED 5
#define RT_ERR_FORMAT 6     // TensorFormatError (ValueError subclass)
#define RT_ERR_NOTFOUND 7   // FileNotFoundError
#define RT_ERR_IO 8         // OSError

typedef int64_t i64;

// One sampled block: P rows per column, Q columns, column-major (row fastest)
// inside the compact buffers at element offset `off`.  Block 0 is the core
// X(I_1..I_n) seen as its mode-1 unfolding (P = |I_1|, Q = prod_{m>=2}|I_m|);
// block k+1 is the mode-(k+1) fiber block C_{k+1} (P = d_{k+1}, Q = |J_{k+1}|).
struct BlockDesc {
  i64 P, Q, off;
  i64 w_off;     // offset of this block's W (Q x r, column-major by q) in a state
  int mode;      // 0-based mode whose factor A maps the rows
  int is_core;
  int r;         // rank of `mode`
  int pad;
};

struct Geom {
  int n;
  int nblk;
  int rank[RT_MAX_MODES];
  i64 dim[RT_MAX_MODES];
  i64 stride[RT_MAX_MODES];      // flat stride of each mode in the FULL tensor
  i64 rstride[RT_MAX_MODES];     // stride of mode m>=1 inside the "rest" offset R (modes 2..n), R stride of mode 0 = 0
  i64 nrows[RT_MAX_MODES];       // |I_k|
  i64 ncols[RT_MAX_MODES];       // |J_k|
  i64 gstride[RT_MAX_MODES];     // strides of G (r_1 x ... x r_n, F-order)
  i64 gsize;                     // prod r
  i64 a_off[RT_MAX_MODES];       // offset of A_k (d_k x r_k col-major) in a state
  i64 state_doubles;             // size of one state (G + A + W)
  BlockDesc blk[RT_MAX_BLOCKS];
  i64 nblk_total;                // sum of P*Q
  const int* stop;               // iteration launches: the engine's stop flag (kernels of an
                                 // iteration enqueued behind one that met the stop rule return at
                                 // once); null for every other launch
};

// An iteration's kernels start with this test: all threads read the same word, so the
// whole grid leaves before any barrier / mbarrier is touched.
__device__ __forceinline__ bool rt_stopped(const int* stop) {
  return stop != nullptr && *reinterpret_cast<const volatile int*>(stop) != 0;
}

// Pointers to the per-mode index data on the device.
struct IndexPtrs {
  const int* rows[RT_MAX_MODES];      // |I_k| sorted 0-based row indices
  const i64* cols[RT_MAX_MODES];      // |J_k| sorted 0-based unfolding columns
  const int* rowpos[RT_MAX_MODES];    // d_k entries: position in I_k or -1
  const i64* colR[RT_MAX_BLOCKS];     // per block column: rest offset R (modes>=2 part)
  const int* coli1[RT_MAX_BLOCKS];    // per block column: mode-1 index (fiber k>=2) or -1
};

__device__ __forceinline__ double ld_elem(const void* p, i64 i, int dtype) {
  return dtype == 0 ? __ldg(reinterpret_cast<const double*>(p) + i)
                    : static_cast<double>(__ldg(reinterpret_cast<const float*>(p) + i));
}

// Strict hard threshold (reference py_kernels.py:226-230: zero iff |x| <= zeta).
__device__ __forceinline__ double hard_thr(double v, double zeta) {
  return fabs(v) <= zeta ? 0.0 : v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree); result valid in every thread.
// `red` must hold blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  __syncthreads();
  return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = red[0];
  for (int w = 1; w < nw; ++w) t = fmax(t, red[w]);
  __syncthreads();
  return t;
}

// Low-rank value of block element (p, q) under a state:
//   l = sum_a A_mode[row(p), a] * W_b[q, a]
// row(p) = p for fiber blocks, I_1[p] for the core block.
__device__ __forceinline__ double eval_low(const double* __restrict__ state, const Geom& g, const BlockDesc& b,
                                           const int* __restrict__ rows0, i64 p, i64 q) {
  const int m = b.mode;
  const i64 d = g.dim[m];
  const i64 row = b.is_core ? (i64)rows0[p] : p;
  const double* A = state + g.a_off[m] + row;
  const double* W = state + b.w_off + q * b.r;
  double acc = 0.0;
  for (int a = 0; a < b.r; ++a) acc = fma(A[a * d], W[a], acc);
  return acc;
}

extern "C" unsigned long long rtcur_launch_counter_add(unsigned long long k);
#define RT_COUNT_LAUNCH() rtcur_launch_counter_add(1ull)
