// full_types.cuh -- arguments of the full-tensor pass K3 (k_full.cu, k_full_tma.cu).
#pragma once
#include "common.cuh"

struct FullArgs {
  const void* X;        // local slab, (hi-lo) x d_2 x ... mode-1 fastest (null: x = 0)
  int dtype;
  i64 lo, hi;           // mode-1 slab
  i64 ncols;            // prod_{m>=2} d_m
  const double* A1;     // d_1 x r_1 col-major (state)
  i64 d1;
  int r1;
  const double* Tf;     // ncols x r_1 row-major
  double zeta;
  void* L;              // optional outputs (dtype), same layout as X
  void* S;
  double* partial;      // [grid][2]
  double* sums;         // [2]: sum (x-L-S)^2, sum x^2
  unsigned int* counter;
};

// TMA-staged K3 (k_full_tma.cu).  Returns 1 when it launched, 0 when the
// geometry is outside its envelope (caller runs the generic k_full), or a
// negative cudaError_t on a launch failure.  `max_grid` bounds the CTA count
// (the partial-sum buffer holds 2*max_grid doubles).
int full_tma_launch(const FullArgs& a, int max_grid, cudaStream_t st);
