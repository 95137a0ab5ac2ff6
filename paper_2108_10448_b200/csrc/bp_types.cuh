// bp_types.cuh -- data layout shared by the block-pass kernels (k_block.cu,
// bp_pass.cuh) and the host planner (engine.cu): tile map, pass arguments,
// shared-memory geometry, TMA/mbarrier helpers.
#pragma once
#include "common.cuh"

// ------------------------------------------------------------------ tile map

#define GATHER_U 4
#define PASS_U 4
#define TILE_MAX_ELEMS 4096
#define BP_X_BYTES 34816     // x bytes per block-pass stage (whole columns)
#define BP_W_DOUBLES 2048    // W doubles per stage and state
#ifndef BP_MIN_CTAS
#define BP_MIN_CTAS 2        // block-pass CTAs per SM (256 threads); 3 measured slower (smaller tiles)
#endif
#define BP_CTA_SMEM (113 * 1024)   // shared-memory budget per CTA (two per SM)

struct TileMap {
  int nblk;
  int tile;                        // max elements per tile
  i64 first[RT_MAX_BLOCKS + 1];    // first tile of each block, first[nblk] = total tiles
  i64 te[RT_MAX_BLOCKS];           // elements per tile of each block (whole columns)
  int cols[RT_MAX_BLOCKS];         // block pass lane mapping: 1 lanes over columns, 0 lanes over rows
  int cpt[RT_MAX_BLOCKS];          // columns per tile (te = cpt * P)
  int ncr[RT_MAX_BLOCKS];          // lanes over rows: column ranges per tile
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

// ------------------------------------------------------------------ K1 block pass

struct PassArgs {
  const void* xb;
  const double* U;         // G pass: U~_1 (|I_1| x r_1 row-major)
  double* t1;              // G pass: r_1 x prod_{m>=2}|I_m| output (F-order)
  int dtype;
  const double* st_s;      // state giving L for the threshold (null: L = 0, first iteration)
  const double* st_e;      // state giving L for the error / trace (null: no error)
  double zeta;
  const double* zetap;     // if set: zeta is read from device memory (graph-captured iterations)
  double* M[RT_MAX_MODES]; // intersection outputs, m_k x p_k column-major (null: skip)
  double* s_out;           // optional sparse values on the blocks
  double* c_out;           // optional clean values
  double* l_out;           // optional low-rank values (state st_e)
  double* partial;         // [tiles][2] per-CTA (e2, x2)
  double* sums;            // [nblk][2]  final (e2, x2)
  unsigned int* counter;   // last-CTA ticket
  int* nonfinite;          // set if a clean intersection entry is not finite
  int want_x2;
  // A pass (AP): per fiber mode k the V_k rows (|J_k| x r row-major) and the
  // per-(block, CTA) partial A rows, reduced by k_areduce_bp
  const double* V[RT_MAX_MODES];
  const double* siginv[RT_MAX_MODES];
  double* apart;
  int ap_grid;             // CTAs of the A-pass launch (partial slot layout)
};

// A pass: CTA owning tile t (relative to the fiber tiles) in a persistent launch of
// G CTAs over N tiles, where CTA c covers [N c / G, N (c + 1) / G)
__host__ __device__ inline long long ap_cta_of(long long t, long long N, long long G) {
  return ((t + 1) * G + N - 1) / N - 1;
}
// partial slot of (block b, CTA c): base_b + (c - first CTA of b) * P_b * r_b doubles
__host__ __device__ inline long long ap_slot(const Geom& g, const TileMap& tm, int G, int b, long long c) {
  const long long N = tm.first[tm.nblk] - tm.first[1];
  long long base = 0;
  for (int bb = 1; bb < b; ++bb) {
    if (tm.first[bb + 1] == tm.first[bb]) continue;   // no tiles (block taken by the fiber pass)
    const long long c0 = ap_cta_of(tm.first[bb] - tm.first[1], N, G);
    const long long c1 = ap_cta_of(tm.first[bb + 1] - 1 - tm.first[1], N, G);
    base += (c1 - c0 + 1) * g.blk[bb].P * g.blk[bb].r;
  }
  const long long cb = ap_cta_of(tm.first[b] - tm.first[1], N, G);
  return base + (c - cb) * g.blk[b].P * g.blk[b].r;
}

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
  int rowmap_ints;   // rowpos staging (ints, >= max fiber-block rows)
  int gp_doubles;    // G-pass cross-warp partials (doubles; 0 for the other passes)
  int a_doubles;     // A rows of a lanes-over-columns block, per state (max P * even pitch)
};

__host__ __device__ inline long long bp_smem_bytes(const BPGeom& G) {
  const long long stage = (long long)G.x_bytes + 2LL * G.w_doubles * 8;
  return (((long long)G.rowmap_ints * 4 + 15) & ~15LL) + (long long)G.gp_doubles * 8 + 2LL * G.a_doubles * 8 +
         (long long)G.stages * stage;
}

