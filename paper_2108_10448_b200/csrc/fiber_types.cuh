// fiber_types.cuh -- interface of the TMA-staged fiber-block pass (k_fiber.cu)
// used by the engine for the threshold and error passes over the fiber blocks.
#pragma once
#include "common.cuh"

struct FiberLaunch {
  Geom g;
  const void* xb;          // compact sampled blocks (dtype)
  int dtype;
  const double* st_s;      // threshold state (null: L = 0, first iteration)
  const double* st_e;      // error state (null: threshold pass)
  double zeta;
  const double* zetap;     // device copy of zeta (graph-captured iterations), or null
  double* M[RT_MAX_MODES]; // threshold pass: intersection outputs (m_k x |J_k| column-major)
  const int* rowpos[RT_MAX_MODES];
  double* partial;         // error pass: [cta][nblk][2] partial sums
  double* sums;            // error pass: [nblk][2]
  unsigned int* counter;
  int* nonfinite;
  // intersection copies X(I_k, J_k) of the fiber blocks (threshold pass input)
  const void* xi;
  i64 xi_off[RT_MAX_MODES];   // element offset of mode k's copy (16-byte aligned)
  i64 xi_ld[RT_MAX_MODES];    // its column stride: |I_k| rounded up to 16 bytes
  const int* rows[RT_MAX_MODES];   // I_k (0-based)
  // A pass (ap != 0): A_k = C_k V_k Sigma_k^+ into a_out (a state), partials in apart
  int ap;
  const double* Vr[RT_MAX_MODES];
  const double* siginv[RT_MAX_MODES];
  double* apart;
  i64 apart_cap;                   // doubles available at apart
  double* a_out;
  unsigned mask;                   // blocks to process (0: every block fiber_pass_blocks takes)
  int reserve_sms;                 // SMs to leave to a kernel this pass runs beside (the eigensolver's CTAs):
                                   // the grid is sized for the rest, so no CTA waits for a second wave
};

// Blocks (bit b = block b) the fiber pass handles for this geometry: fiber
// blocks whose columns are 16-byte aligned in the compact buffer and whose
// rank is <= 16, and (bit 0, error pass only) the core when |I_1| <= 352.
// The rest stay on k_block_pass.
unsigned fiber_pass_blocks(const Geom& g, int dtype);

// Threshold pass (st_e == null: M written, no sums), error pass (st_e set: sums
// of the handled blocks) or A pass (ap set) over the handled fiber blocks.  Returns the
// number of kernels launched or a negative cudaError_t.
int fiber_pass_launch(const FiberLaunch& L, cudaStream_t st);

// Refresh the intersection copies from the compact fiber blocks (after every
// change of the blocks).  Returns 0 or a negative cudaError_t.
int fiber_xi_extract(const FiberLaunch& L, cudaStream_t st);
