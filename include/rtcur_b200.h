/*
 * rtcur_b200.h -- C ABI of the B200-native RTCUR hot path (librtcur_b200.so).
 *
 * Plain pointers, sizes and a cudaStream_t passed as void*; no torch types.
 * Every entry returns an int status (RTCUR_OK = 0); rtcur_last_error() gives
 * the message.  Status -> reference exception mapping used by the Python
 * layer: RTCUR_E_VALUE -> ValueError, RTCUR_E_INDEX -> IndexError,
 * RTCUR_E_ARITH -> ArithmeticError, others -> RuntimeError.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/rtcur):
 *
 *   rtcur_gather_columns   _backend/_core.pyx:265-288  gather_columns(flat, bases, stride, length)
 *   rtcur_hard_threshold   _backend/_core.pyx:252-262  hard_threshold(a, zeta)
 *   rtcur_truncated_svd    linalg.py:59-74 (+ _core.pyx:24-58 dense_svd) truncated_svd(m, r)
 *   rtcur_engine_*         solver.py:260-389 rtcur() loop body:
 *       _absmax            solver.py:184-192  DenseTensorAccessor.inf_norm
 *       _set_sample        fiber_cur.py:148-174 (indices drawn by the host; uploaded here)
 *       _gather            solver.py:234-239 / 172-182  _gather_blocks (core_block, fiber_block)
 *       _iterate           solver.py:324-357  HT on the blocks, assemble_fiber_cur
 *                          (fiber_cur.py:229-274), _eval_blocks (solver.py:242-249),
 *                          sampled_relative_error sums (solver.py:209-231)
 *       _export_*          solver.py:378-389 SolveResult pieces (sparse blocks, FiberCur)
 *   rtcur_full_output      cli.py:237-243 cur_reconstruct_full + hard_threshold(x - L, zeta)
 *
 * Layout: tensors are mode-1-fastest ("F" order, tensor.py:1-10).  Index
 * arrays handed to rtcur_engine_set_sample are the reference's 1-based sorted
 * sets.  Compact blocks are [core (|I_1| x ... x |I_n|, F-order) | fibers
 * C_1 (d_1 x |J_1|, column-major) | ... | C_n].
 */
#ifndef RTCUR_B200_H
#define RTCUR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTCUR_OK 0
#define RTCUR_E_VALUE 1
#define RTCUR_E_INDEX 2
#define RTCUR_E_ARITH 3
#define RTCUR_E_CUDA 4
#define RTCUR_E_UNSUPPORTED 5
#define RTCUR_E_FORMAT 6      /* malformed TNSR file (TensorFormatError) */
#define RTCUR_E_NOTFOUND 7    /* missing file (FileNotFoundError) */
#define RTCUR_E_IO 8          /* other file-system failure (OSError) */

#define RTCUR_F64 0
#define RTCUR_F32 1

typedef struct rtcur_engine rtcur_engine;

const char* rtcur_last_error(void);
const char* rtcur_version(void);
/* number of kernel launches issued by this library since load */
unsigned long long rtcur_launch_count(void);

/* ---- kernel-level plug (reference _backend triple), device pointers, stream-ordered ---- */

/* out (length x ncols, column-major fp64) [i, c] = flat[bases[c] + i * stride] */
int rtcur_gather_columns(const void* flat, int dtype, int64_t flat_len, const int64_t* bases_dev, int64_t ncols,
                         int64_t stride, int64_t length, double* out, void* stream);
/* out[i] = |a[i]| > zeta ? a[i] : 0 */
int rtcur_hard_threshold(const double* a, int64_t n, double zeta, double* out, void* stream);
/* rank-r truncated SVD of an m x p column-major fp64 matrix (min(m, p) <= 235, r <= 32):
 * u (m x r, column-major), s (r, non-increasing), v (p x r, column-major).  Synchronous. */
int rtcur_truncated_svd(const double* m_dev, int64_t m, int64_t p, int r, double* u_dev, double* s_dev,
                        double* v_dev, void* stream);

/* ---- solver engine ---- */

/* Size the device workspace for a problem (bytes); also returns the byte offset
 * and element count of the compact x-block buffer inside it (so a caller can
 * all-reduce it across ranks). */
int rtcur_engine_plan(int n, const int64_t* dims, const int32_t* ranks, const int64_t* row_sizes,
                      const int64_t* col_sizes, int dtype, int64_t* workspace_bytes, int64_t* xblocks_offset,
                      int64_t* xblocks_elems);

/* workspace: device memory of rtcur_engine_plan's size (caller-owned, 256-B aligned).
 * [slab_lo, slab_hi) is this rank's mode-1 slab of X (0, d_1 on one GPU). */
int rtcur_engine_create(rtcur_engine** out, int n, const int64_t* dims, const int32_t* ranks,
                        const int64_t* row_sizes, const int64_t* col_sizes, int dtype, void* workspace,
                        int64_t workspace_bytes, int64_t slab_lo, int64_t slab_hi, void* stream);
int rtcur_engine_destroy(rtcur_engine* e);

/* X (device): this rank's slab, (slab_hi - slab_lo) x d_2 x ... x d_n, mode-1 fastest */
int rtcur_engine_bind(rtcur_engine* e, const void* x_dev);
/* max|X| over the bound slab (K0); synchronous, result on the host */
int rtcur_engine_absmax(rtcur_engine* e, double* out);
/* the same scan split in two: _begin enqueues it on the engine's stream, _end waits
 * and returns max|X| (the host can draw the first sample in between) */
int rtcur_engine_absmax_begin(rtcur_engine* e);
int rtcur_engine_absmax_end(rtcur_engine* e, double* out);
/* Optional copies of X with mode k fastest (rtcur_transpose_mode layout; copies[0]
 * and NULL entries unused): the gather then reads mode-k fibers as contiguous runs
 * instead of stride-prod_{m<k} d_m elements.  Ignored on sharded (slab) engines. */
int rtcur_engine_bind_mode_copies(rtcur_engine* e, const void* const* copies);
/* the same, built by the engine: the mode-k-fastest copy of the bound tensor into `out`
 * (caller-allocated, size of X) on the engine's side stream; the solve's first gather and
 * iteration do not wait for it */
int rtcur_engine_build_mode_copy(rtcur_engine* e, int k, void* out);
/* out = X with mode k moved to the front (then the other modes in order), i.e. for X
 * viewed as (A, d_k, B), out[i + d_k (a + A b)] = X[a + A (i + d_k b)]; dtype 0/1. */
int rtcur_transpose_mode(const void* x, int dtype, int n, const int64_t* dims, int k, void* out, void* stream);
/* rows[k]: |I_k| sorted 1-based indices, cols[k]: |J_k| sorted 1-based unfolding columns (host) */
int rtcur_engine_set_sample(rtcur_engine* e, const int64_t* const* rows, const int64_t* const* cols);
/* gather this rank's owned sampled entries into the compact x blocks (others 0) */
int rtcur_engine_gather(rtcur_engine* e);
/* Mode-1 slab sharding (replaces the reference's in-process
 * _gather_blocks, solver.py:234-239, regathered per RTCUR-R iteration at
 * solver.py:315-322).  bounds: world + 1 slab boundaries of mode 1 (0-based,
 * bounds[rank], bounds[rank+1] = this engine's [lo, hi)).  After set_sample +
 * gather: shard_plan returns each rank's packed entry count (host, world
 * entries); shard_pack writes this rank's owned entries (dtype of X) to send;
 * after an all-gather of the padded segments (recv = world x stride entries),
 * shard_unpack writes every rank's entries into the replicated compact blocks,
 * bit-identical to an unsharded gather. */
int rtcur_engine_set_shards(rtcur_engine* e, int world, int rank, const int64_t* bounds);
int rtcur_engine_shard_plan(rtcur_engine* e, int64_t* counts);
int rtcur_engine_shard_pack(rtcur_engine* e, void* send);
int rtcur_engine_shard_unpack(rtcur_engine* e, const void* recv, int64_t stride);
/* Sample slots: set_sample + gather fill the inactive slot (so they may be enqueued
 * while the previous iteration still runs on the stream); the next iterate_async
 * makes it active.  Workspace byte offset of the compact blocks the next gather
 * writes / the next iteration reads (dtype of X, xblocks_elems entries). */
int rtcur_engine_xblocks_offset(rtcur_engine* e, int64_t* offset);
/* one RTCUR iteration at threshold zeta (already decayed).  first != 0: L = 0.
 * sums (host, 2*(n+1)): per block sum((x-L-S)^2), sum(x^2) of the NEW iterate;
 * flags (host, n): rank-deficiency flags of the new intersections. */
int rtcur_engine_iterate(rtcur_engine* e, double zeta, int first, double* sums, int* flags);
/* the same split in two: enqueue the iteration on the engine's stream and return at once,
 * then wait for it (lets the host draw the next RTCUR-R sample while the GPU works) */
int rtcur_engine_iterate_async(rtcur_engine* e, double zeta, int first);
int rtcur_engine_iterate_wait(rtcur_engine* e, double* sums, int* flags);
/* Speculative pipelining of the stop rule (solver.py:357-358, `if err <= cfg.eps: break`).
 * With a tolerance set (rtcur_engine_set_eps) every iteration ends with a device-side
 * evaluation of the reference's stop test on its own sums; rtcur_engine_last_stop
 * returns it for the iteration waited for last.  When rtcur_engine_can_speculate is 1,
 * iterate_async may be called ONCE more while an iteration is still in flight: the
 * second iteration is enqueued right behind the first, so the stream never idles over
 * the host's round trip; every kernel of an iteration tests the stop flag first, so
 * the second one runs nothing if the first met the stop rule.  iterate_wait always waits for the oldest
 * iteration in flight; after a stop, rtcur_engine_iterate_cancel drops the speculative
 * one and the engine's exportable iterate is again the one that stopped. */
/* start of a solve on a reused engine: the iterate / sample / parity rings restart, so the
 * solve replays the CUDA graphs an earlier solve of this geometry captured */
int rtcur_engine_reset(rtcur_engine* e);
int rtcur_engine_set_eps(rtcur_engine* e, double eps);
int rtcur_engine_can_speculate(rtcur_engine* e);
int rtcur_engine_last_stop(rtcur_engine* e);
int rtcur_engine_iterate_cancel(rtcur_engine* e);

/* Export (device outputs, caller-allocated, fp64), for the iterate of the last
 * rtcur_engine_iterate call:
 *   s_blocks, clean_blocks: N_blk compact sparse values and X - S (either may be NULL)
 *   l_blocks: low-rank values of the new iterate on the blocks (NULL to skip) */
int rtcur_engine_export_blocks(rtcur_engine* e, double* s_blocks, double* clean_blocks, double* l_blocks);
/* per mode k: U_k (|I_k| x r_k), sigma_k (r_k), V_k (|J_k| x r_k), A_k (d_k x r_k), all row-major fp64
 * except A_k (column-major); G (prod r, F-order).  Host pointers; synchronous. */
int rtcur_engine_export_cur(rtcur_engine* e, double* const* U, double* const* sigma, double* const* V,
                            double* const* A, double* G);
/* K3 on the bound slab with the current iterate: optional L/S outputs (dtype of X, slab layout),
 * sums (host, 2): sum((x-L-S)^2), sum(x^2).  Uses a device scratch of prod_{m>=2} d_m * r_1 doubles
 * supplied by the caller (tf_dev). */
int rtcur_engine_full_output(rtcur_engine* e, double zeta, void* L_dev, void* S_dev, double* tf_dev,
                             double* sums);
/* bytes of the tf_dev scratch rtcur_engine_full_output needs */
int64_t rtcur_engine_full_scratch_bytes(rtcur_engine* e);

/* Per-phase device timing with CUDA events on the engine's stream (for the
 * bench roofline).  Phases: 0 absmax (K0), 1 index prep, 2 gather, 3 threshold
 * pass (K1), 4 Gram, 5 eigensolver, 6 SVD post, 7 A pass, 8 G pass, 9 W
 * columns, 10 error pass, 11 export, 12 full output (K3).  nphase >= 13. */
#define RTCUR_NPHASE 13
int rtcur_engine_profile(rtcur_engine* e, int on);
/* Restrict the timers to the phases whose bit (1 << phase) is set in `mask`
 * (default: all).  Timing only the phase a measurement needs keeps the event
 * overhead (two event records per timed phase launch) out of the other phases. */
int rtcur_engine_profile_phases(rtcur_engine* e, uint32_t mask);
/* per-iteration CUDA graphs on (default, unless RTCUR_GRAPHS=0) or off for this engine */
int rtcur_engine_set_graphs(rtcur_engine* e, int on);
int rtcur_engine_profile_read(rtcur_engine* e, double* ms, int64_t* counts, int nphase, int reset);

/* ---- TNSR v1 tensor files (reference tensorfile.py:1-115), streamed disk <-> HBM ----
 * Layout: "TNSR" | u16 version 1 | u16 n | n x u64 extents | prod(extents) f8, mode-1 fastest.
 * rtcur_tnsr_read_header: tensorfile._parse_header (:50-84), plus read_tensor's payload size
 * check (:94-107) when check_payload; messages name the offending byte offset like the
 * reference's TensorFormatError.  dims_cap >= n entries of dims are written.
 * rtcur_tnsr_load: read_tensor (:94-115) into device memory: dtype 0 f64 / 1 f32 (rounded),
 * only mode-1 rows [slab_lo, slab_hi) (slab_hi < 0: all) as a mode-1-fastest slab; the
 * payload streams through pinned double buffers (pread threads || async H2D).  Synchronous.
 * rtcur_tnsr_store: write_tensor (:42-48) from device memory (f64, or f32 widened exactly). */
int rtcur_tnsr_read_header(const char* path, int check_payload, int32_t* version, int32_t* n, int64_t* dims,
                           int dims_cap, int64_t* payload_offset);
int rtcur_tnsr_load(const char* path, int64_t slab_lo, int64_t slab_hi, int dtype, void* dst, void* stream);
int rtcur_tnsr_store(const char* path, int n, const int64_t* dims, int dtype, const void* src, void* stream);

/* Synthetic instance support (bench/tests).  On a mode-1 slab [lo, hi) of a d1 x ... tensor:
 * L(i1, R) = sum_a Y1[i1, a] Tf[R, a] (Y1: d1 x r1 column-major, Tf: ncols x r1 row-major,
 * ncols = prod_{m>=2} d_m, both device pointers shared by every slab).  mode 0 returns
 * sum |L| over the slab in *sum_abs (host, synchronous); mode 1 writes X = L + S (dtype),
 * S Bernoulli(alpha) with values U[-cmu, cmu] keyed by (seed, global element index), so any
 * slab decomposition generates the same tensor bit for bit.  scratch: device, >= 1200 doubles. */
int rtcur_generate_tucker(const double* Y1, const double* Tf, int64_t d1, int r1, int64_t lo, int64_t hi,
                          int64_t ncols, int mode, uint64_t seed, double alpha, double cmu, int dtype, void* X,
                          double* scratch, double* sum_abs, void* stream);

/* Reference-generator outliers (synth.py:101-121, gen_outliers): for k < count,
 * v_k = -mu + (2 mu) * u[k] (numpy Generator.uniform rounding), S[pos[k]] = v_k (S optional),
 * X[pos[k]] += v_k.  X, S fp64 device arrays; pos (0-based, distinct), u device arrays drawn
 * on the host from the reference's exact generator stream. */
int rtcur_scatter_outliers(double* X, const int64_t* pos, const double* u, int64_t count, double mu, double* S,
                           void* stream);
/* sum |x| over n fp64 device values in a fixed order (host result in *out, synchronous);
 * scratch: device, >= 600 doubles.  mu = mean |low| of gen_outliers (synth.py:91-98). */
int rtcur_abs_sum(const double* x, int64_t n, double* scratch, double* out, void* stream);

/* Dense HOSVD alternating projections (reference.py:132-193, the paper's comparison
 * baseline): full-tensor passes of its loop.  rtcur_ap_threshold: S = HT(X - L, zeta)
 * (L may be NULL: L = 0) and C = X - S in one pass.  rtcur_ap_residual: host sums[0] =
 * sum (X - L - S)^2, sums[1] = sum X^2 in a fixed order (synchronous); scratch >= 1200
 * doubles.  All fp64 device arrays of n entries. */
int rtcur_ap_threshold(const double* X, const double* L, int64_t n, double zeta, double* S, double* C, void* stream);
/* max |x| over n device values (dtype 0 f64 / 1 f32; NaN propagates), host result; scratch >= 1 double */
int rtcur_abs_max(const void* x, int dtype, int64_t n, double* scratch, double* out, void* stream);
int rtcur_ap_residual(const double* X, const double* L, const double* S, int64_t n, double* scratch, double* sums,
                      void* stream);

/* Host helper of the index sampler (fiber_cur.py:202-208): append the values of
 * batch not yet marked in seen (population bytes) to out, in first-occurrence
 * order; returns the new length (-1 if a value is out of range). */
int64_t rtcur_append_distinct(int64_t* out, int64_t nout, const int64_t* batch, int64_t nb, unsigned char* seen,
                              int64_t population);
/* The whole iid branch of the reference's without-replacement draw
 * (fiber_cur.py:197-208: batches of need + need//2 + 16 integers(0, population),
 * first occurrences in order, sort(out[:k]) + 1), drawing from a numpy bit
 * generator through its C interface (Generator.bit_generator.ctypes: state
 * address + next_uint32) with numpy's bounded-integer algorithm, so the stream
 * consumed is the one rng.integers would consume.  2 <= population <= 2^32 - 1,
 * 1 <= k < population; seen: (population + 63) / 64 zeroed words (membership
 * bitmap, left zeroed); out: >= 3k + 32 entries.  Returns k (out[0..k) sorted,
 * 1-based) or < 0. */
int64_t rtcur_draw_distinct(void* bitgen_state, void* next_uint32, int64_t population, int64_t k,
                            uint64_t* seen, int64_t* out, int64_t out_cap);

#ifdef __cplusplus
}
#endif
#endif
