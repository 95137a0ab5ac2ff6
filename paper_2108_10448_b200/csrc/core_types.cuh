// core_types.cuh -- interface of the short-column core pass (k_core.cu): the
// G pass (first contraction of the clean core with U~_1) and the core's share
// of the error pass, for cores whose columns (|I_1| rows) are short.
#pragma once
#include "common.cuh"

struct CoreLaunch {
  const void* x;           // the compact core block: |I_1| x Q column-major (dtype), 16-byte aligned
  int dtype;               // 0 fp64, 1 fp32
  int P;                   // |I_1| (rows per column)
  i64 Q;                   // prod_{m>=2} |I_m| (columns)
  int r;                   // r_1
  const int* rows0;        // I_1 (0-based, device)
  i64 dA;                  // d_1: column stride of A_1 in a state
  i64 a_off;               // offset of A_1 in a state
  i64 w_off;               // offset of the core's W rows (Q x r, row-major by column) in a state
  const double* st_s;      // threshold state (L_{k-1}); null: first iteration (L = 0)
  const double* st_e;      // error pass: the new iterate (L_k)
  double zeta;
  const double* zetap;     // device copy of zeta (graph-captured iterations), or null
  int mode;                // 0: G pass (t1 = clean_core^T U~_1), 1: error pass (core sums)
  const double* U;         // G pass: U~_1 (|I_1| x r row-major)
  double* t1;              // G pass: Q x r row-major output
  double* partial;         // error pass: [cta][2]
  double* sums;            // error pass: sums[0] = sum (x - L - S)^2, sums[1] = sum x^2 of the core
  unsigned int* counter;   // error pass: last-CTA ticket
  const int* stop;         // the engine's stop flag (iteration launches), or null
  int nbuf;                // x runs per warp (set by the launcher): 1, or 2 (double-buffered)
};

// The pass applies when a 32-column run of the core is small (32 |I_1| E <= 11 KB,
// so >= 16 warps stay resident per SM) and r_1 <= 8.
bool core_pass_fits(int P, int r, int dtype);

// Launch the pass (G or error mode).  Returns 0 or a negative cudaError_t.
int core_pass_launch(const CoreLaunch& L, cudaStream_t st);
