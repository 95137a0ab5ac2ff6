// engine.cu -- C-ABI entry points (include/rtcur_b200.h) and the per-iteration
// launch schedule of the B200 RTCUR hot path.  One translation unit: the
// kernel files are included so their parameter structs are shared.
//
// Iteration k (reference solver.py:314-375) on the compact sampled blocks:
//   1. k_block_pass  S = HT(X - L_{k-1}, zeta_k), clean intersections -> M_i
//   2. k_gram_*      K_i = B_i B_i^T  (short side of each intersection)
//   3. k_eig         top-r_i eigenbasis of K_i
//   4. k_zproj .. k_complete   rank-r_i truncated SVD (U, sigma, V), pinv cutoff
//   5. A pass (k_block_pass AP) + k_areduce_bp   A_i = C_i V_i S_i^+
//   6. k_gpass/k_modeprod      G = core x_i U_i^T
//   7. k_wcols                 W_b per block column (Tucker evaluation weights)
//   8. k_block_pass  e-sums of X - L_k - S_k and X sums (sampled error)
// States (G, A, W) live in a 3-slot ring so the previous iterate stays
// available for the threshold recomputation and the export.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <atomic>
#include <algorithm>
#include <map>
#include <tuple>

#include "k_block.cu"
#include "k_gram.cu"
#include "k_eig.cu"
#include "k_svdpost.cu"
#include "k_factors.cu"
#include "k_full.cu"
#include "fiber_types.cuh"
#include "core_types.cuh"
#include "../../include/rtcur_b200.h"

static std::atomic<unsigned long long> g_launches{0};
extern "C" unsigned long long rtcur_launch_counter_add(unsigned long long k) { return g_launches.fetch_add(k) + k; }
extern "C" unsigned long long rtcur_launch_count(void) { return g_launches.load(); }

static thread_local std::string g_err;
extern "C" const char* rtcur_last_error(void) { return g_err.c_str(); }
extern "C" const char* rtcur_version(void) { return "rtcur_b200 0.1 sm_100a"; }

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) return fail(RT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define LAUNCH_CHECK()                                                                 \
  do {                                                                                 \
    RT_COUNT_LAUNCH();                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess) return fail(RT_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e) + " @" + std::to_string(__LINE__)); \
  } while (0)

#include "tnsr_io.cu"   // after fail()/CK/LAUNCH_CHECK

static inline i64 cdiv(i64 a, i64 b) { return (a + b - 1) / b; }
static inline i64 align256(i64 x) { return (x + 255) & ~(i64)255; }

// full-storage tridiagonalisation when it fits (faster), else packed
static int eig_pick_full(int s, int r) { return eig_smem_doubles(s, r, 1, 1, 1) <= EIG_SMEM_DOUBLES ? 1 : 0; }
static int eig_pick_nb(int s, int r) {
  // inverse-iteration block: the largest that still leaves room for the warm
  // subspace-iteration scratch (fast path); without it only if nothing fits
  const int full = eig_pick_full(s, r);
  int nb = 0;
  for (int b = 1; b <= r; ++b)
    if (eig_smem_doubles(s, r, b, full, 1) <= EIG_SMEM_DOUBLES) nb = b;
  if (nb == 0)
    for (int b = 1; b <= r; ++b)
      if (eig_smem_doubles(s, r, b, full) <= EIG_SMEM_DOUBLES) nb = b;
  return nb;
}

// k_wcols scratch: the other modes' A rows per thread (max over target modes)
static int wcols_rows_per_thread(const Geom& g) {
  int tot = 0;
  for (int m = 0; m < g.n; ++m) tot += g.rank[m];
  int mn = g.rank[0];
  for (int m = 0; m < g.n; ++m) mn = std::min(mn, g.rank[m]);
  return std::max(1, tot - mn);
}
static int wcols_smem(const Geom& g) { return (int)((g.gsize + 128 * wcols_rows_per_thread(g)) * 8); }

#define BP_GRID (148 * 2)   // persistent block-pass CTAs (2 per SM)

static int rbucket(int r) { return r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : 32; }

#define DISPATCH_R(RB, KERNEL, GRID, BLOCK, SMEM, STREAM, ...)                     \
  do {                                                                               \
    switch (RB) {                                                                    \
      case 4: KERNEL<4><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;           \
      case 8: KERNEL<8><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;           \
      case 16: KERNEL<16><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;         \
      default: KERNEL<32><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;         \
    }                                                                                \
  } while (0)

#define RT_SAMPLE_SLOTS 3  // sample ring: the running iteration's, the next one's (staged), the one being staged
#define RT_STATE_SLOTS 6   // iterate ring: latest, its threshold state, a shadow, the speculative pair + 1

struct Plan {
  Geom g;
  TileMap tm;
  TileMap tm_gp;   // G pass: the core block's tiles (lanes over columns when possible)
  TileMap tm_core; // threshold/error passes on k_block_pass: the blocks the fiber pass does not take
  TileMap tm_thr;  // threshold pass on k_block_pass: only fiber blocks (the core yields nothing there)
  unsigned fiber_mask;   // blocks handled by the TMA fiber pass (k_fiber.cuh)
  unsigned fb_thr, fb_ap, fb_err;   // per pass (RTCUR_FB_PASSES bits 1/2/4 switch passes off for A/B runs)
  bool core_k;                      // the core's G pass and error pass on k_core_pass (short columns)
  i64 o_cpart;                      // its per-CTA error partials
  TileMap tm_ap;   // A pass on k_block_pass: the fiber blocks the fiber pass does not take
  i64 xi_off[RT_MAX_MODES], xi_ld[RT_MAX_MODES];   // intersection copies (elements) inside o_xi
  i64 o_xi;
  i64 o_fapart, fapart_cap;   // fiber-pass A-pass partials
  i64 res_bytes;              // sums | flags | non-finite flag (contiguous from o_sums)
  int dtype;
  int esize;
  int rmax, rb;
  i64 s[RT_MAX_MODES], l[RT_MAX_MODES];
  int tall[RT_MAX_MODES];
  int nb[RT_MAX_MODES];
  bool lug[RT_MAX_MODES];   // inverse-iteration LU in global scratch (o_lug)
  i64 col_off[RT_MAX_BLOCKS + 1];
  int gram_maxchunks, gram_maxpairs, gram_cl;
  i64 dmax, lmax, smax, qmax;
  i64 g_tmp;         // doubles per G temp buffer
  i64 w_tmp;         // doubles per W-chain temp buffer
  int hchunk, h_maxchunks;
  BPGeom bp;
  BPGeom bp_gp;
  BPGeom bp_ap;    // A pass: the pass tiles' stages + a per-block P x r accumulator
  int ap_grid, ap_threads;
  i64 o_apart2;
  // workspace offsets (bytes)
  i64 o_rows[RT_MAX_MODES], o_cols[RT_MAX_MODES], o_rowpos, o_colR, o_coli1, o_coloff;
  i64 o_zeta;       // device copy of the iteration's threshold (graph-captured iterations read it)
  i64 samp_delta;   // bytes from sample slot 0 (index sets, maps, compact blocks) to slot 1
  i64 o_Kfull[RT_MAX_MODES];
  i64 o_xb, o_state, o_M[RT_MAX_MODES], o_gpart, o_K[RT_MAX_MODES], o_hv[RT_MAX_MODES], o_E[RT_MAX_MODES], o_lug[RT_MAX_MODES],
      o_lam[RT_MAX_MODES], o_Z[RT_MAX_MODES], o_hpart[RT_MAX_MODES], o_H[RT_MAX_MODES], o_Q[RT_MAX_MODES],
      o_U[RT_MAX_MODES], o_V[RT_MAX_MODES], o_sig[RT_MAX_MODES], o_siginv[RT_MAX_MODES], o_perm[RT_MAX_MODES],
      o_degen[RT_MAX_MODES], o_flags, o_nonfinite, o_counters, o_absmax, o_gt0, o_gt1, o_bpart, o_sums,
      o_fpart, o_dbg, o_fast, o_wt0, o_wt1, o_wt0s, o_wt1s;
  i64 res_stride;             // bytes between the two (launch-parity) copies of the result range
  i64 total;
};

static int make_plan(Plan& P, int n, const int64_t* dims, const int32_t* ranks, const int64_t* row_sizes,
                     const int64_t* col_sizes, int dtype) {
  memset(&P, 0, sizeof(P));
  if (n < 1 || n > RT_MAX_MODES) return fail(RT_ERR_UNSUPPORTED, "number of modes must be in [1, 8]");
  if (dtype != 0 && dtype != 1) return fail(RT_ERR_VALUE, "dtype must be RTCUR_F64 or RTCUR_F32");
  Geom& g = P.g;
  g.n = n;
  g.nblk = n + 1;
  P.dtype = dtype;
  P.esize = dtype == 0 ? 8 : 4;
  i64 total = 1;
  for (int m = 0; m < n; ++m) {
    if (dims[m] < 1) return fail(RT_ERR_VALUE, "nonpositive extent");
    g.dim[m] = dims[m];
    g.stride[m] = total;
    total *= dims[m];
  }
  i64 rs = 0;
  for (int m = 0; m < n; ++m) {
    g.rstride[m] = (m == 0) ? 0 : (m == 1 ? 1 : rs);
    if (m >= 1) rs = (m == 1 ? dims[1] : rs * dims[m]);
  }
  g.gsize = 1;
  P.rmax = 1;
  for (int m = 0; m < n; ++m) {
    const i64 rest = total / dims[m];
    if (ranks[m] < 1 || ranks[m] > dims[m]) return fail(RT_ERR_VALUE, "rank outside [1, d_k]");
    if (row_sizes[m] < 1 || row_sizes[m] > dims[m]) return fail(RT_ERR_VALUE, "row sample size outside [1, d_k]");
    if (col_sizes[m] < 1 || col_sizes[m] > rest) return fail(RT_ERR_VALUE, "column sample size outside range");
    if (ranks[m] > row_sizes[m] || ranks[m] > col_sizes[m])
      return fail(RT_ERR_VALUE, "mode " + std::to_string(m + 1) + ": rank exceeds sample sizes");
    if (ranks[m] > RT_MAX_RANK) return fail(RT_ERR_UNSUPPORTED, "rank > 32 not supported");
    g.rank[m] = ranks[m];
    g.nrows[m] = row_sizes[m];
    g.ncols[m] = col_sizes[m];
    g.gstride[m] = g.gsize;
    g.gsize *= ranks[m];
    P.rmax = std::max(P.rmax, (int)ranks[m]);
    P.s[m] = std::min(row_sizes[m], col_sizes[m]);
    P.l[m] = std::max(row_sizes[m], col_sizes[m]);
    P.tall[m] = row_sizes[m] > col_sizes[m];
    if (P.s[m] > 235) return fail(RT_ERR_UNSUPPORTED, "intersection short side > 235 not supported");
  }
  if (g.gsize > 8192) return fail(RT_ERR_UNSUPPORTED, "prod(ranks) > 8192 not supported");
  P.rb = rbucket(P.rmax);
  // blocks
  i64 off = 0;
  {
    BlockDesc& b = g.blk[0];
    b.P = row_sizes[0];
    b.Q = 1;
    for (int m = 1; m < n; ++m) b.Q *= row_sizes[m];
    b.off = off;
    b.mode = 0;
    b.is_core = 1;
    b.r = ranks[0];
    off += b.P * b.Q;
  }
  for (int k = 0; k < n; ++k) {
    BlockDesc& b = g.blk[k + 1];
    b.P = dims[k];
    b.Q = col_sizes[k];
    off = (off + 3) & ~(i64)3;   // 16-byte aligned block start (TMA bulk copies)
    b.off = off;
    b.mode = k;
    b.is_core = 0;
    b.r = ranks[k];
    off += b.P * b.Q;
  }
  g.nblk_total = off;
  // state layout: G | A_0..A_{n-1} | W_0..W_n
  i64 so = align256(g.gsize * 8) / 8;
  for (int m = 0; m < n; ++m) {
    g.a_off[m] = so;
    so += align256(dims[m] * ranks[m] * 8) / 8;
  }
  for (int b = 0; b < g.nblk; ++b) {
    g.blk[b].w_off = so;
    so += align256(g.blk[b].Q * g.blk[b].r * 8) / 8;
  }
  g.state_doubles = so;
  // tiles
  TileMap& tm = P.tm;
  tm.nblk = g.nblk;
  // Block-pass tiles: whole columns, at most xb bytes of x per stage.  Lanes
  // over columns when >= 32 columns fit (32 * 2^k columns, <= 8 column groups),
  // else lanes over rows.  xb starts at BP_X_BYTES and shrinks until two stages
  // (plus the staged A rows and the G pass's partials) leave two CTAs per SM.
  {
    i64 maxP = 1;
    for (int b = 0; b < g.nblk; ++b) maxP = std::max(maxP, g.blk[b].P);
    if (maxP > TILE_MAX_ELEMS) return fail(RT_ERR_UNSUPPORTED, "mode extent above 4096 not supported");
    BPGeom& G = P.bp;
    tm.tile = TILE_MAX_ELEMS;
    for (i64 xb = BP_X_BYTES;; xb = std::max<i64>(maxP * P.esize, xb * 3 / 4)) {
      G.rowmap_ints = (int)maxP;
      G.gp_doubles = 0;
      G.stages = 3;
      i64 xmax = 16;   // largest tile's x bytes (the stage's x region)
      int wmax = 2;
      i64 amax = 0;
      i64 t = 0;
      for (int b = 0; b < g.nblk; ++b) {
        tm.first[b] = t;
        const i64 Pb = g.blk[b].P, nel = Pb * g.blk[b].Q;
        const int rb = g.blk[b].r;
        const i64 xcap = std::max<i64>(1, xb / (Pb * P.esize));
        const i64 wcap = std::max<i64>(1, (BP_W_DOUBLES - 4) / rb);
        i64 cpt;
        if (std::min(xcap, wcap) >= 32) {
          cpt = 32;
          while (cpt * 2 <= std::min<i64>(std::min(xcap, wcap), 256)) cpt *= 2;
          tm.cols[b] = 1;
        } else {
          cpt = std::min(xcap, wcap);
          tm.cols[b] = 0;
        }
        tm.ncr[b] = 1;
        tm.te[b] = cpt * Pb;
        tm.cpt[b] = (int)cpt;
        xmax = std::max<i64>(xmax, cpt * Pb * P.esize);
        if (tm.cols[b]) amax = std::max<i64>(amax, Pb * ((rb + 1) & ~1));
        wmax = std::max(wmax, (int)(cpt * rb + 4));
        t += cdiv(nel, tm.te[b]);
      }
      tm.first[g.nblk] = t;
      G.x_bytes = (int)(((xmax + 15) & ~15LL) + 32);
      G.w_doubles = (wmax + 1) & ~1;
      G.a_doubles = (int)((amax + 1) & ~1);
      // three stages when two CTAs per SM still fit (with the G pass's partials), else two
      BPGeom gg = G;
      gg.gp_doubles = 256 * P.rmax;
      if (bp_smem_bytes(gg) + 1024 > BP_CTA_SMEM) G.stages = 2;
      gg.stages = G.stages;
      if (bp_smem_bytes(gg) + 1024 <= BP_CTA_SMEM || xb <= std::max<i64>(4096, maxP * P.esize)) break;
    }
    // G pass: its own map over the core block only, lanes over columns (32 * 2^k
    // columns within BP_X_BYTES) with the staged A/U rows and partials; cols = 0
    // when not even 32 columns fit (the warp-per-column k_gpass runs instead)
    {
      TileMap& tg = P.tm_gp;
      tg = tm;
      BPGeom& Gg = P.bp_gp;
      const i64 Pc = g.blk[0].P;
      const int rc = g.blk[0].r;
      const i64 xcap = std::max<i64>(1, (i64)BP_X_BYTES / (Pc * P.esize));
      const i64 wcap = std::max<i64>(1, (BP_W_DOUBLES - 4) / rc);
      i64 cpt = std::min(xcap, wcap);
      tg.cols[0] = cpt >= 32 ? 1 : 0;
      if (tg.cols[0]) {
        i64 c2 = 32;
        while (c2 * 2 <= std::min<i64>(cpt, 256)) c2 *= 2;
        cpt = c2;
      }
      tg.cpt[0] = (int)cpt;
      tg.te[0] = cpt * Pc;
      tg.first[0] = 0;
      tg.first[1] = cdiv(Pc * g.blk[0].Q, tg.te[0]);
      Gg.rowmap_ints = 16;
      Gg.x_bytes = (int)(((cpt * Pc * P.esize + 15) & ~15LL) + 32);
      Gg.w_doubles = (int)((cpt * rc + 4 + 1) & ~1);
      Gg.a_doubles = (int)((Pc * ((rc + 1) & ~1) + 1) & ~1);
      Gg.gp_doubles = 256 * rc;
      Gg.stages = bp_smem_bytes(BPGeom{3, Gg.x_bytes, Gg.w_doubles, 16, Gg.gp_doubles, Gg.a_doubles}) + 1024 <= BP_CTA_SMEM
                      ? 3
                      : 2;
    }
    // A pass over the fiber tiles of the pass map
    {
      BPGeom& Ga = P.bp_ap;
      Ga = G;
      Ga.a_doubles = 0;
      Ga.gp_doubles = 2;
      for (int b = 1; b < g.nblk; ++b) Ga.gp_doubles = (int)std::max<i64>(Ga.gp_doubles, g.blk[b].P * g.blk[b].r);
      Ga.gp_doubles = (Ga.gp_doubles + 1) & ~1;
      Ga.stages = 3;
      if (bp_smem_bytes(Ga) + 1024 > BP_CTA_SMEM) Ga.stages = 2;
      const i64 nt = tm.first[g.nblk] - tm.first[1];
      // two 256-thread CTAs per SM when they fit, else one 512-thread CTA (16 warps either way)
      P.ap_threads = bp_smem_bytes(Ga) + 1024 <= BP_CTA_SMEM ? 256 : 512;
      P.ap_grid = (int)std::max<i64>(1, std::min<i64>(P.ap_threads == 256 ? 296 : 148, nt));
    }
  }

  // fiber blocks on the TMA fiber pass; k_block_pass keeps the core (and any block outside its envelope)
  P.fiber_mask = fiber_pass_blocks(g, dtype);
  {
    const char* fp = getenv("RTCUR_FB_PASSES");
    const int bits = fp ? atoi(fp) : 7;
    P.fb_thr = (bits & 1) ? P.fiber_mask & ~1u : 0u;
    P.fb_ap = (bits & 2) ? P.fiber_mask & ~1u : 0u;
    P.fb_err = (bits & 4) ? P.fiber_mask : 0u;
    // short core columns: the core's G pass and error share on k_core_pass -- opt-in
    // (RTCUR_CORE_PASS=1): measured +2 % at config 4, -3 % at config 0 against the
    // block pass / fiber pass, so the default keeps those
    const char* cpv = getenv("RTCUR_CORE_PASS");
    P.core_k = (cpv && cpv[0] == '1') && core_pass_fits((int)g.blk[0].P, g.rank[0], dtype) && g.blk[0].Q >= 64;
    if (P.core_k) P.fb_err &= ~1u;
  }
  {
    TileMap& tc = P.tm_core;
    tc = P.tm;
    i64 t = 0;
    for (int b = 0; b < g.nblk; ++b) {
      const i64 nt = P.tm.first[b + 1] - P.tm.first[b];
      tc.first[b] = t;
      if (!(P.fb_err >> b & 1) && !(b == 0 && P.core_k)) t += nt;
    }
    tc.first[g.nblk] = t;
    TileMap& ta = P.tm_ap;
    ta = P.tm;
    t = 0;
    for (int b = 0; b < g.nblk; ++b) {
      const i64 nt = P.tm.first[b + 1] - P.tm.first[b];
      ta.first[b] = t;
      if (!(P.fb_ap >> b & 1)) t += nt;
    }
    ta.first[g.nblk] = t;
    // threshold pass: M_k comes from fiber blocks only; the core's clean values are
    // recomputed by the G pass, so k_block_pass needs no core tiles there
    TileMap& tt = P.tm_thr;
    tt = P.tm;
    t = 0;
    for (int b = 0; b < g.nblk; ++b) {
      const i64 nt = P.tm.first[b + 1] - P.tm.first[b];
      tt.first[b] = t;
      if (b > 0 && !(P.fb_thr >> b & 1)) t += nt;
    }
    tt.first[g.nblk] = t;
  }

  P.col_off[0] = 0;
  for (int b = 0; b < g.nblk; ++b) P.col_off[b + 1] = P.col_off[b] + g.blk[b].Q;
  // gram / svd sizing
  P.gram_maxchunks = 1;
  P.gram_maxpairs = 1;
  P.dmax = 1;
  P.lmax = 1;
  P.smax = 1;
  P.qmax = 1;
  // split-K so that the Gram tiles fill ~4 waves of 148 SMs
  {
    int pairs_tot = 0;
    i64 lm = 1;
    for (int m = 0; m < n; ++m) {
      const int nt = (int)cdiv(P.s[m], GRAM_T);
      pairs_tot += nt * (nt + 1) / 2;
      lm = std::max(lm, P.l[m]);
    }
    // split-K over ~6 waves of CTAs (measured: the tile loop is latency-bound, so more
    // CTAs in flight beat fewer split-K partials)
    const char* gw = getenv("RTCUR_GRAM_WAVES");
    const char* gm = getenv("RTCUR_GRAM_MIN_CL");
    const i64 waves = gw ? std::max(1, atoi(gw)) : 6;
    const i64 mincl = gm ? std::max(GRAM_KS, atoi(gm)) : GRAM_KS;
    const i64 want = std::max<i64>(1, cdiv(waves * 148, pairs_tot));
    P.gram_cl = (int)std::max<i64>(std::min<i64>(mincl, cdiv(lm, GRAM_KS) * GRAM_KS),
                                   cdiv(cdiv(lm, want), GRAM_KS) * GRAM_KS);
    if (!gw && !gm) {
      // wave-quantised choice: the DMMA tile kernel runs 3 CTAs per SM (168
      // registers x 128 threads, 34.8 KB static shared memory); minimise
      // ceil(CTAs / (3 x 148)) x (chunk length + a fixed per-CTA cost of ~32
      // columns) over chunk lengths in k-steps (a 2.03-wave grid costs 3 waves)
      const i64 slots = 3 * 148, c0 = 32;
      i64 best = -1, bcl = P.gram_cl;
      for (i64 cl = GRAM_KS; cl <= cdiv(lm, GRAM_KS) * GRAM_KS; cl += GRAM_KS) {
        i64 ctas = 0;
        for (int m = 0; m < n; ++m) {
          const i64 nt = cdiv(P.s[m], GRAM_T);
          ctas += nt * (nt + 1) / 2 * cdiv(P.l[m], cl);
        }
        const i64 cost = cdiv(ctas, slots) * (cl + c0);
        if (best < 0 || cost <= best) { best = cost; bcl = cl; }   // ties: longer chunks, fewer partials
      }
      P.gram_cl = (int)bcl;
    }
  }
  for (int m = 0; m < n; ++m) {
    const int nt = (int)cdiv(P.s[m], GRAM_T);
    P.gram_maxpairs = std::max(P.gram_maxpairs, nt * (nt + 1) / 2);
    P.gram_maxchunks = std::max(P.gram_maxchunks, (int)cdiv(P.l[m], P.gram_cl));
    P.dmax = std::max(P.dmax, (i64)dims[m]);
    P.lmax = std::max(P.lmax, P.l[m]);
    P.smax = std::max(P.smax, P.s[m]);
    // inverse-iteration batch: as many LU factorisations as fit in 227 KB next to K and E
    int nb = eig_pick_nb((int)P.s[m], ranks[m]);
    if (nb < 1) return fail(RT_ERR_UNSUPPORTED, "intersection too large for the shared-memory eigensolver");
    P.nb[m] = nb;
  }
  for (int b = 0; b < g.nblk; ++b) P.qmax = std::max(P.qmax, g.blk[b].Q);
  P.hchunk = HG_CH;
  P.h_maxchunks = (int)cdiv(P.lmax, P.hchunk);
  // G temporaries: largest partially contracted core
  {
    i64 mx = 1, cur = ranks[0];
    for (int m = 1; m < n; ++m) cur *= row_sizes[m];
    mx = cur;
    for (int m = 1; m < n; ++m) {
      cur = cur / row_sizes[m] * ranks[m];
      mx = std::max(mx, cur);
    }
    P.g_tmp = std::max<i64>(mx, g.gsize);
    // W_core chain G x_2 A_2(I_2) .. x_n A_n(I_n): intermediates (r1, I2..Im, r_{m+1}..rn), m < n
    i64 wmx = 1;
    for (int m = 1; m + 1 < n; ++m) {
      i64 sz = ranks[0];
      for (int l = 1; l <= m; ++l) sz *= row_sizes[l];
      for (int l = m + 1; l < n; ++l) sz *= ranks[l];
      wmx = std::max(wmx, sz);
    }
    // same for the full-tensor chain (K3 weights): (r1, d2..dm, r_{m+1}..rn)
    for (int m = 1; m + 1 < n; ++m) {
      i64 sz = ranks[0];
      for (int l = 1; l <= m; ++l) sz *= dims[l];
      for (int l = m + 1; l < n; ++l) sz *= ranks[l];
      wmx = std::max(wmx, sz);
    }
    P.w_tmp = wmx;
  }
  // workspace carve
  i64 o = 0;
  auto take = [&](i64 bytes) { i64 r = o; o += align256(std::max<i64>(bytes, 8)); return r; };
  // sample slot 0 (index sets, row/column maps, compact blocks); slot 1 follows at samp_delta
  const i64 samp0 = o;
  for (int m = 0; m < n; ++m) P.o_rows[m] = take(row_sizes[m] * 4);
  for (int m = 0; m < n; ++m) P.o_cols[m] = take(col_sizes[m] * 8);
  {
    i64 sd = 0;
    for (int m = 0; m < n; ++m) sd += dims[m];
    P.o_rowpos = take(sd * 4);
  }
  P.o_colR = take(P.col_off[g.nblk] * 8);
  P.o_coli1 = take(P.col_off[g.nblk] * 4);
  P.o_coloff = take((RT_MAX_BLOCKS + 1) * 8);
  P.o_xb = take(g.nblk_total * P.esize + 64);   // +64: aligned bulk-copy supersets may read past the end
  {
    // intersection copies X(I_k, J_k) of the fiber blocks for the fiber pass's threshold
    const i64 va = 16 / P.esize;
    i64 xo = 0;
    for (int m = 0; m < n; ++m) {
      P.xi_ld[m] = (row_sizes[m] + va - 1) / va * va;
      P.xi_off[m] = xo;
      xo += (P.xi_ld[m] * col_sizes[m] + va - 1) / va * va;
    }
    P.o_xi = take(P.fiber_mask ? xo * P.esize + 64 : 8);
  }
  P.samp_delta = o - samp0;
  for (int s = 1; s < RT_SAMPLE_SLOTS; ++s) take(P.samp_delta - 8);   // slots 1.. (aligned like slot 0)
  P.o_state = take((i64)RT_STATE_SLOTS * g.state_doubles * 8);
  P.o_zeta = take(64);   // per launch parity p, at +32 p: zeta | eps; the stop flag at +16
  for (int m = 0; m < n; ++m) P.o_M[m] = take(row_sizes[m] * col_sizes[m] * 8);
  P.o_gpart = take((i64)n * P.gram_maxchunks * P.gram_maxpairs * GRAM_T * GRAM_T * 8);
  for (int m = 0; m < n; ++m) {
    const i64 s = P.s[m];
    P.o_K[m] = take(s * (s + 1) / 2 * 8);
    P.o_Kfull[m] = take(s > 128 ? s * s * 8 : 8);   // mirrored copy for the packed-storage Lanczos matvec
    P.o_E[m] = take(s * ranks[m] * 8);
    {
      // RTCUR_EIG_LU_GLOBAL=1 forces the global-scratch LU (tests), =0 disables it
      static const int lug_env = [] { const char* v = getenv("RTCUR_EIG_LU_GLOBAL"); return v ? atoi(v) : -1; }();
      P.lug[m] = lug_env == 1 || (lug_env != 0 && P.nb[m] < ranks[m]);
      P.o_lug[m] = take(P.lug[m] ? s * ranks[m] * 4 * 8 + s * ranks[m] : 8);
    }
    P.o_lam[m] = take(ranks[m] * 8);
    P.o_Z[m] = take(P.l[m] * ranks[m] * 8);
    P.o_hpart[m] = take((i64)cdiv(P.l[m], HG_CH) * ranks[m] * (ranks[m] + 1) / 2 * 8);
    P.o_H[m] = take(ranks[m] * ranks[m] * 8);
    P.o_Q[m] = take(ranks[m] * ranks[m] * 8);
    P.o_U[m] = take(row_sizes[m] * ranks[m] * 8);
    P.o_V[m] = take(col_sizes[m] * ranks[m] * 8);
    P.o_sig[m] = take(ranks[m] * 8);
    P.o_siginv[m] = take(ranks[m] * 8);
    P.o_perm[m] = take(ranks[m] * 4);
    P.o_degen[m] = take((ranks[m] + 1) * 4);
  }
  // the iteration's results in one contiguous range (one D2H per iteration):
  // sums (2 nblk doubles) | flags (n ints, padded to 8 bytes) | non-finite flag
  {
    P.res_stride = align256(2 * g.nblk * 8 + ((n * 4 + 7) & ~7LL) + 8);
    const i64 res0 = take(2 * P.res_stride);   // one copy per launch parity (an iteration's error
                                               // pass may run under the next iteration's eigensolver)
    P.o_sums = res0;
    P.o_flags = res0 + 2 * g.nblk * 8;
    P.o_nonfinite = P.o_flags + ((n * 4 + 7) & ~7LL);
    P.res_bytes = 2 * g.nblk * 8 + ((n * 4 + 7) & ~7LL) + 8;   // (+ the stop flag's copy)
  }
  P.o_counters = take(64 * 4);
  P.o_absmax = take(8);
  {
    // A-pass partials: one P_b x r_b slot per (fiber block, CTA that touches it)
    // (for the full pass map and for the map without the fiber pass's blocks)
    auto slots = [&](const TileMap& tmx) {
      const i64 N = tmx.first[P.g.nblk] - tmx.first[1];
      i64 tot = 0;
      for (int b = 1; b < P.g.nblk; ++b) {
        if (N <= 0 || tmx.first[b + 1] == tmx.first[b]) continue;
        const i64 G = std::max<i64>(1, std::min<i64>(P.ap_grid, N));   // (run_factors' grid)
        const i64 c0 = ap_cta_of(tmx.first[b] - tmx.first[1], N, G);
        const i64 c1 = ap_cta_of(tmx.first[b + 1] - 1 - tmx.first[1], N, G);
        tot += (c1 - c0 + 1) * P.g.blk[b].P * P.g.blk[b].r;
      }
      return tot;
    };
    P.o_apart2 = take(std::max<i64>(1, std::max(slots(P.tm), slots(P.tm_ap))) * 8);
  }
  P.o_gt0 = take(P.g_tmp * 8);
  P.o_gt1 = take(P.g_tmp * 8);
  P.o_wt0 = take(P.w_tmp * 8);
  P.o_wt1 = take(P.w_tmp * 8);
  P.o_wt0s = take(P.w_tmp * 8);   // the side stream's W chain (shadow state, concurrent with the iteration's)
  P.o_wt1s = take(P.w_tmp * 8);
  P.o_bpart = take((i64)BP_GRID * g.nblk * 2 * 8 + 64);
  P.o_cpart = take(2 * 148 * 8 * 8 + 64);
  {
    // fiber-pass A pass: one d_k x r_k slot per (fiber block, CTA touching it) -- at most 296 + n slots
    i64 mx = 1;
    // (column offsets per CTA x rows <= max(d_k, 352 threads x 4 rows))
    for (int m = 0; m < n; ++m) mx = std::max<i64>(mx, std::max<i64>(dims[m], 1408) * ranks[m]);
    P.fapart_cap = P.fiber_mask ? (148 * 2 + n) * mx : 1;   // (up to two CTAs per SM, k_fiber.cuh)
    P.o_fapart = take(P.fapart_cap * 8);
  }
  P.o_fpart = take(148 * 8 * 2 * 8);
  P.o_dbg = take(8 * RT_MAX_MODES * 8);
  P.o_fast = take(RT_MAX_MODES * 4);
  P.total = o;
  return RT_OK;
}

// profiled phases (index into rtcur_engine_profile_read outputs)
enum { PH_ABSMAX = 0, PH_PREP, PH_GATHER, PH_THRESH, PH_GRAM, PH_EIG, PH_SVDPOST, PH_APASS, PH_GPASS, PH_WCOLS,
       PH_ERROR, PH_EXPORT, PH_FULL, RT_NPHASE };

struct ProfPair {
  int ph;
  cudaEvent_t b, e;
  bool owned;   // from the engine's event pool (returned at flush)
  unsigned seq; // iteration launch it belongs to (0: outside an iteration)
};
// An iteration is captured as a short list of graph segments.  A segment ends where
// the stream needs an event between graphs: the begin / end of a profiled phase, or
// the point where the eigensolver starts (eig_ev: the side-stream prefetch of the next
// sample waits for it).  (Gating the segments with conditional IF nodes on the stop
// flag was measured at ~50 us per iteration on B200 -- more than the host round trip
// it hides -- so the kernels test the flag themselves, Geom::stop / rt_stopped.)
enum { CUT_NONE = 0, CUT_PROF_BEGIN, CUT_PROF_END,
       CUT_EIG,     // the eigensolver starts: record eig_ev, enqueue the previous iteration's tail under it
       CUT_JOIN,    // the eigensolver is enqueued: wait for that tail (its stop flag) before the SVD post
       CUT_STATE }; // G and A of the new iterate are complete: record st_ev (the shadow's W waits for it)
struct GraphSeg {
  cudaGraphExec_t exec = nullptr;   // null: nothing was captured before the cut
  int cut = CUT_NONE, ph = 0;       // event to record after the segment
};
struct GraphEntry {
  std::vector<GraphSeg> segs;        // threshold ... column weights of the new iterate
  std::vector<GraphSeg> tail;        // error pass, stop rule, result copy
  std::vector<ProfPair> prof, prof_tail;   // event-record nodes of the profiled phases (graph-owned events)
  unsigned long long nkernels = 0;   // kernel launches captured in segs (counted at every replay)
  unsigned long long nk_tail = 0;    // ... in tail
};

struct ShardState;   // shard_xchg.cu

struct rtcur_engine {
  Plan P;
  char* ws;
  cudaStream_t st;
  i64 lo, hi;
  const void* X;
  const void* mcopy[RT_MAX_MODES];   // optional mode-k-fastest copies of X (rtcur_engine_bind_mode_copies)
  int cur;          // ring slot of the latest iterate (-1: none)
  int act, stg;     // sample slots: active (iterations, exports) and staged (next set_sample/gather), -1: none
  int sample_epoch; // bumped whenever a staged sample becomes active
  int w_epoch[RT_STATE_SLOTS];   // sample epoch each slot's W (column weights) was built for
  // RTCUR-R shadow: slot `shadow` holds a copy of state `shadow_of` (G, A) whose W was
  // evaluated on the sample staged for epoch `shadow_epoch` (side stream, under the running
  // iteration): the next iteration thresholds against it instead of re-evaluating in place,
  // so the running iterate stays intact for its error pass and for the exports
  int shadow, shadow_of, shadow_epoch;
  int alloc_rr;     // ring cursor of the state-slot allocator
  int cur_par;      // parity of the launch being enqueued / captured (result range, control words)
  bool wt_alt;      // W-chain scratch: the side stream's pair
  // The tail of an iteration (error pass, stop rule, result copy) does not feed the next
  // iteration's threshold / Gram / eigensolver: it is held back and enqueued on `tail`
  // under the NEXT iteration's eigensolver (3-4 CTAs on an otherwise idle GPU); that
  // iteration joins it before its SVD post, the first kernel that must see the stop flag.
  cudaStream_t tail;
  struct TailRef { struct GraphEntry* ge; int par; unsigned seq; bool valid; } tail_pending;
  int tail_reserve;       // SMs the held-back tail's error pass leaves to the eigensolver it runs beside
  cudaEvent_t svd_ev;     // recorded when an iteration's SVD post starts (after its eigensolver and the join)
  cudaEvent_t st_ev;      // the running iteration's G and A are complete (the shadow's W waits for it)
  unsigned st_ev_seq;     // launch that recorded st_ev last
  cudaEvent_t main_ev;    // the running iteration's main part is enqueued up to here
  bool mcopy_fresh;       // mode copies being built on the side stream (mcopy_ev), not yet ordered with st
  cudaEvent_t mcopy_ev;
  bool r_mode;            // samples are re-staged between iterations (RTCUR-R): cut the graph at CUT_STATE
  unsigned cur_of_seq;    // launch that produced the latest iterate
  cudaEvent_t tl_base;    // diagnostics: recorded at a solve's first iteration (RTCUR_PROF_TIMELINE)
  bool join_needed;       // the iteration being launched must wait for join_ev before its SVD post
  cudaEvent_t join_ev;
  int npending;     // iterate_async calls awaiting their iterate_wait (2: one speculative)
  bool use_fast;    // allow the warm-started subspace-iteration eigensolver
  cudaEvent_t done[2];   // recorded after the iteration's result copies (by launch parity)
  int par;          // parity of the next launch: pinned zeta / result slot, done event
  int pend_par[2];  // parities of the launches in flight, oldest first
  int last_stop;    // stop flag the device computed for the iteration waited for last
  double eps;       // stop tolerance of the device-side stop rule (<= 0: never stops)
  // speculation (rtcur_engine_iterate_async while one iteration is in flight): the
  // bookkeeping before the speculative launch, restored by rtcur_engine_iterate_cancel
  bool spec_ok;     // speculative launches allowed (RTCUR_SPEC=0 disables them)
  struct Snap {
    int cur, prev, act, stg, sample_epoch, w_epoch[RT_STATE_SLOTS], shadow, shadow_of, shadow_epoch, alloc_rr;
    double zeta_last;
    bool xi_valid[RT_SAMPLE_SLOTS];
  } snap;
  bool snap_valid;
  unsigned launch_seq, cur_seq, snap_seq;   // iteration launches so far; the one being enqueued; the speculative one
  int prev;         // ring slot of the one before (-1: none, i.e. latest is iteration 1)
  double zeta_last;
  bool sampled;
  char* h_export;    // page-locked staging of rtcur_engine_export_cur (grown on demand)
  size_t h_export_bytes;
  double* h_pinned;  // host staging: sums, flags
  int* h_flags;
  i64* h_idx;        // pinned staging for index upload (one half per sample slot)
  i64 h_idx_len;
  cudaEvent_t idx_ev[RT_SAMPLE_SLOTS];   // H2D of each slot's index staging done
  // optional per-phase CUDA-event timing (rtcur_engine_profile)
  bool prof_on;
  unsigned prof_mask;  // phases timed while prof_on
  double prof_ms[RT_NPHASE];
  long long prof_cnt[RT_NPHASE];
  std::vector<cudaEvent_t>* prof_pool;
  std::vector<ProfPair>* prof_pending;
  cudaEvent_t prof_open[RT_NPHASE];
  // per-iteration CUDA graphs (rtcur_engine_iterate_async): one per launch-shape key
  bool use_graphs;
  bool capturing;
  cudaStream_t cap_st;             // private stream the iteration is captured on
  cudaStream_t cap_st2;            // second capture stream: a parallel branch inside the iteration's graph
  cudaEvent_t fork_ev, join2_ev;   // its fork / join (captured as graph edges)
  std::map<unsigned long long, GraphEntry>* graphs;
  GraphEntry* cap_entry;
  std::vector<GraphSeg>* cap_segs; // the list the capture appends to (cap_entry->segs or ->tail)
  int cap_err;                     // first error inside a capture cut (prof_begin/prof_end are void)
  const double* zetap_cur;         // device zeta while an iteration body is enqueued/captured
  bool xi_valid[RT_SAMPLE_SLOTS];  // the sample slot's intersection copies match its blocks
  cudaEvent_t absmax_ev;           // rtcur_engine_absmax_begin's D2H done
  bool absmax_pending;
  ShardState* shard;               // mode-1 slab exchange plan (rtcur_engine_set_shards), or null
  // RTCUR-R prefetch: a sample staged while an iteration is in flight (set_sample +
  // gather) runs on a side stream, concurrently with that iteration (its eigensolver
  // occupies a few SMs); the side stream first waits for pre_ev (everything enqueued
  // before the running iteration: the last readers of the slot being refilled) and
  // the next iteration waits for side_ev.  RTCUR_SIDE_PREFETCH=0 keeps it in order.
  bool use_side;
  bool staging_on_side;
  cudaStream_t side;
  cudaEvent_t pre_ev, side_ev;
  cudaEvent_t eig_ev;              // recorded inside the iteration when its eigensolver starts:
                                   // the prefetch waits for it, so it overlaps k_eig (few SMs)
                                   // rather than the wide threshold / Gram kernels before it
  template <typename T> T* at(i64 off) const { return reinterpret_cast<T*>(ws + off); }
  double* state(int slot) const { return at<double>(P.o_state) + (i64)slot * P.g.state_doubles; }
  i64 roff() const { return (i64)cur_par * P.res_stride; }   // this launch's copy of the result range
  i64 sd(int slot) const { return (i64)slot * P.samp_delta; }   // byte shift of a sample slot
  int act_slot() const { return act >= 0 ? act : 0; }
  char* xb(int slot) const { return ws + P.o_xb + sd(slot); }
};

static cudaEvent_t prof_event(rtcur_engine* e) {
  if (!e->prof_pool->empty()) {
    cudaEvent_t ev = e->prof_pool->back();
    e->prof_pool->pop_back();
    return ev;
  }
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  return ev;
}
// ---- graph segments (see GraphSeg)
// the device control words: [zeta (double) | eps (double) | stop (int)] at o_zeta
static inline int* stop_flag(const rtcur_engine* e) { return e->at<int>(e->P.o_zeta + 16); }

static cudaError_t seg_begin(rtcur_engine* e) {
  return cudaStreamBeginCapture(e->cap_st, cudaStreamCaptureModeThreadLocal);
}

// close the segment being captured: instantiate it (unless empty) and note the event
// the stream records after it
static cudaError_t seg_end(rtcur_engine* e, int cut, int ph) {
  cudaGraph_t cap = nullptr;
  cudaError_t ce = cudaStreamEndCapture(e->cap_st, &cap);
  GraphSeg sg;
  sg.cut = cut;
  sg.ph = ph;
  if (ce == cudaSuccess && cap) {
    size_t nn = 0;
    ce = cudaGraphGetNodes(cap, nullptr, &nn);
    if (ce == cudaSuccess && nn > 0) ce = cudaGraphInstantiate(&sg.exec, cap, 0);
  }
  if (cap) cudaGraphDestroy(cap);
  if (ce == cudaSuccess) e->cap_segs->push_back(sg);
  return ce;
}

static void cap_cut(rtcur_engine* e, int cut, int ph) {
  if (e->cap_err != (int)cudaSuccess) return;
  cudaError_t ce = seg_end(e, cut, ph);
  if (ce == cudaSuccess) ce = seg_begin(e);
  e->cap_err = (int)ce;
}

static void prof_begin(rtcur_engine* e, int ph) {
  if (!e->prof_on || !((e->prof_mask >> ph) & 1u)) return;
  if (e->capturing) {   // an event-record node inside the segment (events owned by the graph entry)
    cudaEvent_t ev = nullptr;
    if (cudaEventCreate(&ev) == cudaSuccess &&
        cudaEventRecordWithFlags(ev, e->st, cudaEventRecordExternal) == cudaSuccess)
      e->prof_open[ph] = ev;
    return;
  }
  cudaEvent_t ev = prof_event(e);
  cudaEventRecord(ev, e->st);
  e->prof_open[ph] = ev;
}
static void prof_end(rtcur_engine* e, int ph) {
  if (!e->prof_on) return;
  if (e->capturing) {
    if (!e->prof_open[ph]) return;
    cudaEvent_t ev = nullptr;
    if (cudaEventCreate(&ev) == cudaSuccess &&
        cudaEventRecordWithFlags(ev, e->st, cudaEventRecordExternal) == cudaSuccess)
      (e->cap_segs == &e->cap_entry->tail ? e->cap_entry->prof_tail : e->cap_entry->prof)
          .push_back({ph, e->prof_open[ph], ev, false, 0u});
    e->prof_open[ph] = nullptr;
    return;
  }
  if (!e->prof_open[ph]) return;
  cudaEvent_t ev = prof_event(e);
  cudaEventRecord(ev, e->st);
  e->prof_pending->push_back({ph, e->prof_open[ph], ev, true, e->cur_seq});
  e->prof_open[ph] = nullptr;
}
// the tail of iteration `t` (error pass, stop rule, result copy) on `st`, then its done event
static int launch_tail(rtcur_engine* e, const rtcur_engine::TailRef& t, cudaStream_t st) {
  for (auto& sg : t.ge->tail) {
    if (sg.exec) CK(cudaGraphLaunch(sg.exec, st));
    if (sg.cut == CUT_PROF_BEGIN) {
      cudaEvent_t ev = prof_event(e);
      CK(cudaEventRecord(ev, st));
      e->prof_open[sg.ph] = ev;
    } else if (sg.cut == CUT_PROF_END && e->prof_open[sg.ph]) {
      cudaEvent_t ev = prof_event(e);
      CK(cudaEventRecord(ev, st));
      e->prof_pending->push_back({sg.ph, e->prof_open[sg.ph], ev, true, t.seq});
      e->prof_open[sg.ph] = nullptr;
    }
  }
  for (auto p : t.ge->prof_tail) {
    p.seq = t.seq;
    e->prof_pending->push_back(p);
  }
  rtcur_launch_counter_add(t.ge->nk_tail);
  CK(cudaEventRecord(e->done[t.par], st));
  return RT_OK;
}

// a held-back tail goes out in stream order (nothing will run over it)
static int flush_tail(rtcur_engine* e) {
  if (!e->tail_pending.valid) return RT_OK;
  const rtcur_engine::TailRef t = e->tail_pending;
  e->tail_pending.valid = false;
  return launch_tail(e, t, e->st);
}

// replay a captured iteration's main part: its segments with the events between them
static int launch_entry(rtcur_engine* e, GraphEntry& ge) {
  cudaStream_t cs = e->st;
  for (auto& sg : ge.segs) {
    if (sg.exec) CK(cudaGraphLaunch(sg.exec, cs));
    if (sg.cut == CUT_PROF_BEGIN) {
      cudaEvent_t ev = prof_event(e);
      CK(cudaEventRecord(ev, cs));
      e->prof_open[sg.ph] = ev;
    } else if (sg.cut == CUT_PROF_END && e->prof_open[sg.ph]) {
      cudaEvent_t ev = prof_event(e);
      CK(cudaEventRecord(ev, cs));
      e->prof_pending->push_back({sg.ph, e->prof_open[sg.ph], ev, true, e->cur_seq});
      e->prof_open[sg.ph] = nullptr;
    } else if (sg.cut == CUT_EIG) {
      CK(cudaEventRecord(e->eig_ev, e->st));
      if (e->tail_pending.valid) {   // the previous iteration's tail runs under this eigensolver
        const rtcur_engine::TailRef t = e->tail_pending;
        e->tail_pending.valid = false;
        CK(cudaStreamWaitEvent(e->tail, e->eig_ev, 0));
        if (int st = launch_tail(e, t, e->tail)) return st;
        e->join_needed = true;
        e->join_ev = e->done[t.par];
      }
    } else if (sg.cut == CUT_JOIN) {
      if (e->join_needed) CK(cudaStreamWaitEvent(e->st, e->join_ev, 0));
      e->join_needed = false;
      CK(cudaEventRecord(e->svd_ev, e->st));   // the SVD post starts (see rtcur_engine_set_sample)
    } else if (sg.cut == CUT_STATE) {
      CK(cudaEventRecord(e->st_ev, e->st));
      e->st_ev_seq = e->cur_seq;
    }
  }
  for (auto p : ge.prof) {
    p.seq = e->cur_seq;
    e->prof_pending->push_back(p);
  }
  return RT_OK;
}
// after a stream synchronisation: fold the completed intervals into the totals;
// intervals still in flight (work enqueued behind the synchronisation point, e.g.
// a prefetched gather) stay pending
static void prof_flush(rtcur_engine* e) {
  std::vector<ProfPair> keep;
  for (auto& p : *e->prof_pending) {
    if (cudaEventQuery(p.e) != cudaSuccess) {
      keep.push_back(p);
      continue;
    }
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.b, p.e) == cudaSuccess) {
      e->prof_ms[p.ph] += ms;
      e->prof_cnt[p.ph] += 1;
      // diagnostics (RTCUR_PROF_TIMELINE=1): where each profiled interval sits, relative to
      // the solve's first iteration, on whichever stream ran it
      static const bool tl = getenv("RTCUR_PROF_TIMELINE") != nullptr;
      float t0 = 0.f;
      if (tl && e->tl_base && cudaEventElapsedTime(&t0, e->tl_base, p.b) == cudaSuccess)
        fprintf(stderr, "TL seq %u phase %d start_us %.1f dur_us %.1f\n", p.seq, p.ph, 1e3f * t0, 1e3f * ms);
    }
    if (p.owned) {
      e->prof_pool->push_back(p.b);
      e->prof_pool->push_back(p.e);
    }
  }
  e->prof_pending->swap(keep);
}

#include "shard_xchg.cu"   // after prof_begin/prof_end, fail()/CK/LAUNCH_CHECK

static int set_smem_limits_once() {
  // function attributes are per device context: once per device
  static std::atomic<int> done[RT_MAX_DEVICES];
  int dev = 0, optin = 227 * 1024;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= RT_MAX_DEVICES) return fail(RT_ERR_VALUE, "device ordinal out of range");
  if (done[dev].load()) return RT_OK;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // per kernel: opt-in maximum minus its static shared memory
#define SMEM_ATTR(F)                                                                          \
  do {                                                                                        \
    cudaFuncAttributes fa;                                                                    \
    CK(cudaFuncGetAttributes(&fa, F));                                                        \
    CK(cudaFuncSetAttribute(F, cudaFuncAttributeMaxDynamicSharedMemorySize,                   \
                            optin - (int)fa.sharedSizeBytes));                                \
  } while (0)
  SMEM_ATTR(k_eig);
  SMEM_ATTR(k_wcols<4>); SMEM_ATTR(k_wcols<8>); SMEM_ATTR(k_wcols<16>); SMEM_ATTR(k_wcols<32>);
  SMEM_ATTR((k_wcols_warp<4, 32>)); SMEM_ATTR((k_wcols_warp<8, 32>)); SMEM_ATTR((k_wcols_warp<16, 32>));
  SMEM_ATTR((k_wcols_warp<32, 32>));
  SMEM_ATTR((k_wcols_warp<4, 8>)); SMEM_ATTR((k_wcols_warp<8, 8>)); SMEM_ATTR((k_wcols_warp<16, 8>));
  SMEM_ATTR((k_wcols_warp<32, 8>));
  SMEM_ATTR(k_zproj<4>); SMEM_ATTR(k_zproj<8>); SMEM_ATTR(k_zproj<16>); SMEM_ATTR(k_zproj<32>);
#define BP_ATTRS(RB)                                                                                     \
  SMEM_ATTR((k_block_pass<true, true, false, true, false, RB, false>));                                  \
  SMEM_ATTR((k_block_pass<true, false, false, true, false, RB, false>));                                 \
  SMEM_ATTR((k_block_pass<false, true, false, true, false, RB, false>));                                 \
  SMEM_ATTR((k_block_pass<false, false, false, true, false, RB, false>));                                \
  SMEM_ATTR((k_block_pass<true, false, true, false, false, RB, false>));                                 \
  SMEM_ATTR((k_block_pass<false, false, true, false, false, RB, false>));                                \
  SMEM_ATTR((k_block_pass<true, true, false, false, false, RB, false>));                                 \
  SMEM_ATTR((k_block_pass<false, true, false, false, false, RB, false>));                                \
  SMEM_ATTR((k_block_pass<true, false, false, false, true, RB, false>));                                 \
  SMEM_ATTR((k_block_pass<false, false, false, false, true, RB, false>));                                \
  SMEM_ATTR((k_block_pass<true, false, false, false, false, RB, true>));                                 \
  SMEM_ATTR((k_block_pass<false, false, false, false, false, RB, true>))
  BP_ATTRS(4); BP_ATTRS(8); BP_ATTRS(16); BP_ATTRS(32);
#undef BP_ATTRS
  SMEM_ATTR(k_hgram<1>); SMEM_ATTR(k_hgram<2>); SMEM_ATTR(k_hgram<3>);
#undef SMEM_ATTR
  // L2 fetch granularity for the sampled gathers (element-sized loads scattered
  // over X): RTCUR_L2_FETCH=<32|64|128> bytes; unset leaves the device default
  if (const char* gf = getenv("RTCUR_L2_FETCH")) {
    const int b = atoi(gf);
    if (b == 32 || b == 64 || b == 128) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)b));
  }
  done[dev].store(1);
  return RT_OK;
}

static IndexPtrs make_ip_slot(const rtcur_engine* e, int slot) {
  const Plan& P = e->P;
  const i64 d = e->sd(slot);
  IndexPtrs ip;
  memset(&ip, 0, sizeof(ip));
  i64 roff = 0;
  for (int m = 0; m < P.g.n; ++m) {
    ip.rows[m] = e->at<int>(P.o_rows[m] + d);
    ip.cols[m] = e->at<i64>(P.o_cols[m] + d);
    ip.rowpos[m] = e->at<int>(P.o_rowpos + d) + roff;
    roff += P.g.dim[m];
  }
  for (int b = 0; b < P.g.nblk; ++b) {
    ip.colR[b] = e->at<i64>(P.o_colR + d) + P.col_off[b];
    ip.coli1[b] = e->at<int>(P.o_coli1 + d) + P.col_off[b];
  }
  return ip;
}
// the active sample (iterations, exports, K3)
static IndexPtrs make_ip(const rtcur_engine* e) { return make_ip_slot(e, e->act_slot()); }

// the warm-started fast path needs extra scratch; used only when it fits
static int eig_fast_ok(const Plan& P, int m) {
  const int s = (int)P.s[m], r = P.g.rank[m];
  return !P.tall[m] && eig_smem_doubles(s, r, P.nb[m], eig_pick_full(s, r), 1) <= EIG_SMEM_DOUBLES;
}
static int eig_smem_bytes(const Plan& P, int m) {
  const int s = (int)P.s[m], r = P.g.rank[m];
  return (int)(eig_smem_doubles(s, r, P.nb[m], eig_pick_full(s, r), eig_fast_ok(P, m)) * 8);
}

extern "C" int rtcur_engine_plan(int n, const int64_t* dims, const int32_t* ranks, const int64_t* row_sizes,
                                 const int64_t* col_sizes, int dtype, int64_t* workspace_bytes,
                                 int64_t* xblocks_offset, int64_t* xblocks_elems) {
  Plan* P = new Plan;
  int st = make_plan(*P, n, dims, ranks, row_sizes, col_sizes, dtype);
  if (st == RT_OK) {
    if (workspace_bytes) *workspace_bytes = P->total;
    if (xblocks_offset) *xblocks_offset = P->o_xb;
    if (xblocks_elems) *xblocks_elems = P->g.nblk_total;
  }
  delete P;
  return st;
}

extern "C" int rtcur_engine_create(rtcur_engine** out, int n, const int64_t* dims, const int32_t* ranks,
                                   const int64_t* row_sizes, const int64_t* col_sizes, int dtype, void* workspace,
                                   int64_t workspace_bytes, int64_t slab_lo, int64_t slab_hi, void* stream) {
  rtcur_engine* e = new rtcur_engine;
  memset((void*)e, 0, sizeof(*e));
  int st = make_plan(e->P, n, dims, ranks, row_sizes, col_sizes, dtype);
  if (st != RT_OK) { delete e; return st; }
  if (workspace_bytes < e->P.total || workspace == nullptr) { delete e; return fail(RT_ERR_VALUE, "workspace too small"); }
  if (((uintptr_t)workspace & 255) != 0) { delete e; return fail(RT_ERR_VALUE, "workspace must be 256-byte aligned"); }
  if (slab_lo < 0 || slab_hi > dims[0] || slab_lo >= slab_hi) { delete e; return fail(RT_ERR_VALUE, "bad mode-1 slab"); }
  e->ws = (char*)workspace;
  e->st = (cudaStream_t)stream;
  e->lo = slab_lo;
  e->hi = slab_hi;
  e->cur = e->prev = e->shadow = -1;
  e->act = e->stg = -1;
  for (int m = 0; m < RT_MAX_MODES; ++m) e->mcopy[m] = nullptr;
  for (int s = 0; s < RT_SAMPLE_SLOTS; ++s) e->idx_ev[s] = nullptr;
  e->prof_mask = ~0u;
  e->use_fast = getenv("RTCUR_NO_FAST_EIG") == nullptr;
  e->prof_pool = new std::vector<cudaEvent_t>();
  if (cudaEventCreateWithFlags(&e->done[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->done[1], cudaEventDisableTiming) != cudaSuccess) {
    delete e;
    return fail(RT_ERR_CUDA, "cudaEventCreate");
  }
  {
    const char* sv = getenv("RTCUR_SPEC");
    e->spec_ok = !(sv && sv[0] == '0');
  }
  e->prof_pending = new std::vector<ProfPair>();
  e->graphs = new std::map<unsigned long long, GraphEntry>();
  // on by default (config 1: 2099 -> 2236 iters/s once the fiber pass added launches);
  // RTCUR_GRAPHS=0 launches every kernel on the stream
  {
    const char* gv = getenv("RTCUR_GRAPHS");
    e->use_graphs = !(gv && gv[0] == '0');
  }
  e->capturing = false;
  e->cap_entry = nullptr;
  e->zetap_cur = nullptr;
  if (cudaStreamCreateWithFlags(&e->cap_st, cudaStreamNonBlocking) != cudaSuccess) {
    delete e;
    return fail(RT_ERR_CUDA, "cudaStreamCreate");
  }
  if (cudaStreamCreateWithFlags(&e->cap_st2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->join2_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete e;
    return fail(RT_ERR_CUDA, "cudaStreamCreate");
  }
  cudaError_t ce = cudaMallocHost(&e->h_pinned, 4096);
  if (ce != cudaSuccess) { delete e; return fail(RT_ERR_CUDA, "cudaMallocHost"); }
  e->h_flags = reinterpret_cast<int*>(e->h_pinned + 256);
  // per sample slot: the byte span of the device index range (rows + cols with the carve's padding)
  const i64 idx_span = e->P.o_cols[n - 1] + col_sizes[n - 1] * 8 - e->P.o_rows[0];
  e->h_idx_len = (idx_span + 7) / 8;
  ce = cudaMallocHost(&e->h_idx, RT_SAMPLE_SLOTS * (e->h_idx_len * 8 + 64));
  if (ce != cudaSuccess) { cudaFreeHost(e->h_pinned); delete e; return fail(RT_ERR_CUDA, "cudaMallocHost"); }
  // counters + col offsets
  CK(cudaMemsetAsync(e->ws + e->P.o_counters, 0, 64 * 4, e->st));
  // zero the compact blocks once: the alignment pads between blocks are never
  // written by the gather and must not carry garbage into rank all-reduces
  for (int s = 0; s < RT_SAMPLE_SLOTS; ++s) CK(cudaMemsetAsync(e->xb(s), 0, e->P.g.nblk_total * e->P.esize + 64, e->st));
  for (int s = 0; s < RT_SAMPLE_SLOTS; ++s) CK(cudaEventCreateWithFlags(&e->idx_ev[s], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->absmax_ev, cudaEventDisableTiming));
  {
    // on by default (with the speculative pipeline: config 1 +5 %, config 4 +12 %,
    // DESIGN.md §6); RTCUR_SIDE_PREFETCH=0 keeps the staging in stream order
    const char* sv = getenv("RTCUR_SIDE_PREFETCH");
    e->use_side = !(sv && sv[0] == '0');
  }
  CK(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&e->pre_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->side_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->eig_ev, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&e->tail, cudaStreamNonBlocking));

  CK(cudaEventCreateWithFlags(&e->st_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->main_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->mcopy_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->svd_ev, cudaEventDisableTiming));
  CK(cudaMemcpyAsync(e->ws + e->P.o_coloff, e->P.col_off, sizeof(i64) * (RT_MAX_BLOCKS + 1), cudaMemcpyHostToDevice, e->st));
  CK(cudaStreamSynchronize(e->st));
  // opt-in shared memory: kernel attributes are process-global, so raise every
  // dynamic-smem kernel to the device maximum once (pooled engines of different
  // geometries share them; occupancy follows the bytes of each launch)
  {
    int st = set_smem_limits_once();
    if (st) { delete e; return st; }
  }
  *out = e;
  return RT_OK;
}

extern "C" int rtcur_engine_destroy(rtcur_engine* e) {
  if (!e) return RT_OK;
  cudaStreamSynchronize(e->st);
  shard_free(e);
  if (e->h_pinned) cudaFreeHost(e->h_pinned);
  if (e->h_export) cudaFreeHost(e->h_export);
  if (e->h_idx) cudaFreeHost(e->h_idx);
  for (int s = 0; s < 2; ++s)
    if (e->done[s]) cudaEventDestroy(e->done[s]);
  if (e->absmax_ev) cudaEventDestroy(e->absmax_ev);
  for (int s = 0; s < RT_SAMPLE_SLOTS; ++s)
    if (e->idx_ev[s]) cudaEventDestroy(e->idx_ev[s]);
  if (e->prof_pending) {
    for (auto& p : *e->prof_pending)
      if (p.owned) {
        cudaEventDestroy(p.b);
        cudaEventDestroy(p.e);
      }
    delete e->prof_pending;
  }
  if (e->graphs) {
    for (auto& kv : *e->graphs) {
      for (auto* v : {&kv.second.segs, &kv.second.tail})
        for (auto& sg : *v)
          if (sg.exec) cudaGraphExecDestroy(sg.exec);
      for (auto* v : {&kv.second.prof, &kv.second.prof_tail})
        for (auto& p : *v) {
          cudaEventDestroy(p.b);
          cudaEventDestroy(p.e);
        }
    }
    delete e->graphs;
  }
  if (e->cap_st) cudaStreamDestroy(e->cap_st);
  if (e->cap_st2) cudaStreamDestroy(e->cap_st2);
  if (e->fork_ev) cudaEventDestroy(e->fork_ev);
  if (e->join2_ev) cudaEventDestroy(e->join2_ev);
  if (e->side) cudaStreamSynchronize(e->side), cudaStreamDestroy(e->side);
  if (e->pre_ev) cudaEventDestroy(e->pre_ev);
  if (e->side_ev) cudaEventDestroy(e->side_ev);
  if (e->eig_ev) cudaEventDestroy(e->eig_ev);
  if (e->tail) cudaStreamSynchronize(e->tail), cudaStreamDestroy(e->tail);
  if (e->st_ev) cudaEventDestroy(e->st_ev);
  if (e->main_ev) cudaEventDestroy(e->main_ev);
  if (e->mcopy_ev) cudaEventDestroy(e->mcopy_ev);
  if (e->svd_ev) cudaEventDestroy(e->svd_ev);
  if (e->prof_pool) {
    for (auto ev : *e->prof_pool) cudaEventDestroy(ev);
    delete e->prof_pool;
  }
  delete e;
  return RT_OK;
}

// Start of a solve on a (pooled) engine: every ring -- iterate slots, sample slots, launch
// parity -- restarts from zero, so each solve walks the same sequence of launch shapes and
// replays the graphs the first solve of this geometry captured (a solve that started where
// the previous one left off kept meeting new slot combinations: tens of milliseconds of
// capture + instantiation each, for many solves).
extern "C" int rtcur_engine_reset(rtcur_engine* e) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  if (e->npending) return fail(RT_ERR_VALUE, "iteration in flight");
  if (int st = flush_tail(e)) return st;
  e->cur = e->prev = e->shadow = -1;
  e->act = e->stg = -1;
  e->alloc_rr = 0;
  e->par = 0;
  e->cur_par = 0;
  e->snap_valid = false;
  e->r_mode = false;
  e->join_needed = false;
  e->sampled = false;
  e->sample_epoch = 0;
  for (int i = 0; i < RT_STATE_SLOTS; ++i) e->w_epoch[i] = -1;
  for (int s = 0; s < RT_SAMPLE_SLOTS; ++s) e->xi_valid[s] = false;
  if (e->staging_on_side) {   // (a staged sample the previous solve never used)
    CK(cudaStreamWaitEvent(e->st, e->side_ev, 0));
    e->staging_on_side = false;
  }
  return RT_OK;
}

extern "C" int rtcur_engine_bind(rtcur_engine* e, const void* x_dev) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  e->X = x_dev;   // NULL unbinds (K3 then reconstructs L only)
  return RT_OK;
}

extern "C" int rtcur_engine_bind_mode_copies(rtcur_engine* e, const void* const* copies) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  if (e->mcopy_fresh) {   // copies still being built on the side stream: whatever reuses their
    CK(cudaStreamWaitEvent(e->st, e->mcopy_ev, 0));   // memory on this stream comes after
    e->mcopy_fresh = false;
  }
  for (int m = 0; m < RT_MAX_MODES; ++m) e->mcopy[m] = (copies && m < e->P.g.n && m > 0) ? copies[m] : nullptr;
  return RT_OK;
}

extern "C" int rtcur_transpose_mode(const void* x, int dtype, int n, const int64_t* dims, int k, void* out,
                                    void* stream);

// Build the mode-k-fastest copy of the bound tensor into `out` on the engine's side stream
// and let the gathers that follow it there read mode-k fibers contiguously.  The solve's
// first gather and iteration do not wait for it (that gather reads strided fibers once):
// the copies (2 x 233 us at config 1) leave the solve's start-up path.
extern "C" int rtcur_engine_build_mode_copy(rtcur_engine* e, int k, void* out) {
  if (!e || !e->X) return fail(RT_ERR_VALUE, "no tensor bound");
  if (k < 1 || k >= e->P.g.n || !out) return fail(RT_ERR_VALUE, "bad mode copy");
  if (!(e->lo == 0 && e->hi == e->P.g.dim[0])) return fail(RT_ERR_VALUE, "mode copies need the whole tensor");
  cudaStream_t st = e->use_side ? e->side : e->st;
  if (st != e->st) {
    CK(cudaEventRecord(e->pre_ev, e->st));        // X is complete on the solve's stream
    CK(cudaStreamWaitEvent(st, e->pre_ev, 0));
  }
  int64_t dims[RT_MAX_MODES];
  for (int m = 0; m < e->P.g.n; ++m) dims[m] = e->P.g.dim[m];
  if (int rc = rtcur_transpose_mode(e->X, e->P.dtype, e->P.g.n, dims, k, out, st)) return rc;
  e->mcopy[k] = out;
  if (st != e->st) {
    CK(cudaEventRecord(e->mcopy_ev, st));
    e->mcopy_fresh = true;
  }
  return RT_OK;
}

extern "C" int rtcur_transpose_mode(const void* x, int dtype, int n, const int64_t* dims, int k, void* out,
                                    void* stream) {
  if (!x || !out || !dims || n < 1 || k < 0 || k >= n || (dtype != 0 && dtype != 1))
    return fail(RT_ERR_VALUE, "bad transpose arguments");
  i64 A = 1, B = 1;
  for (int m = 0; m < k; ++m) A *= dims[m];
  for (int m = k + 1; m < n; ++m) B *= dims[m];
  const i64 dk = dims[k];
  const dim3 grid((unsigned)cdiv(A, 32), (unsigned)cdiv(dk, 32), (unsigned)std::min<i64>(B, 65535));
  if (grid.x > 0x7fffffff || grid.y > 65535) return fail(RT_ERR_UNSUPPORTED, "transpose grid too large");
  if (dtype == 0)
    k_transpose_mode<double><<<grid, 256, 0, (cudaStream_t)stream>>>((const double*)x, A, dk, B, (double*)out);
  else
    k_transpose_mode<float><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)x, A, dk, B, (float*)out);
  LAUNCH_CHECK();
  return RT_OK;
}

// zeta_0 = max|X| in two halves: _begin enqueues the scan and its 8-byte D2H
// (pinned slot 240), _end waits for it -- the host draws the first sample in
// between.  rtcur_engine_absmax = begin + end.
extern "C" int rtcur_engine_absmax_begin(rtcur_engine* e) {
  if (!e || !e->X) return fail(RT_ERR_VALUE, "no tensor bound");
  const Plan& P = e->P;
  i64 nloc = e->hi - e->lo;
  for (int m = 1; m < P.g.n; ++m) nloc *= P.g.dim[m];
  unsigned long long* d = e->at<unsigned long long>(P.o_absmax);
  CK(cudaMemsetAsync(d, 0, 8, e->st));
  prof_begin(e, PH_ABSMAX);
  int nsm = 148;
  const int grid = nsm * 8;
  if (P.dtype == 0) k_absmax<double><<<grid, 256, 0, e->st>>>((const double*)e->X, nloc, d);
  else k_absmax<float><<<grid, 256, 0, e->st>>>((const float*)e->X, nloc, d);
  LAUNCH_CHECK();
  prof_end(e, PH_ABSMAX);
  CK(cudaMemcpyAsync(e->h_pinned + 240, d, 8, cudaMemcpyDeviceToHost, e->st));
  CK(cudaEventRecord(e->absmax_ev, e->st));
  e->absmax_pending = true;
  return RT_OK;
}

extern "C" int rtcur_engine_absmax_end(rtcur_engine* e, double* out) {
  if (!e || !e->absmax_pending) return fail(RT_ERR_VALUE, "no abs-max scan in flight");
  CK(cudaEventSynchronize(e->absmax_ev));
  e->absmax_pending = false;
  prof_flush(e);
  unsigned long long bits;
  memcpy(&bits, e->h_pinned + 240, 8);
  double v;
  memcpy(&v, &bits, 8);
  *out = v;
  return RT_OK;
}

extern "C" int rtcur_engine_absmax(rtcur_engine* e, double* out) {
  if (int st = rtcur_engine_absmax_begin(e)) return st;
  return rtcur_engine_absmax_end(e, out);
}

// Is an iteration's tail held back and run under the next eigensolver?  (RTCUR_TAIL_DEFER=0|1
// overrides.)  Always for RTCUR-F; for RTCUR-R only while the sampled blocks are small --
// there the next sample's gather already runs under the eigensolver, and at config 4 (87 MB
// of blocks, a 116 us gather against a 72 us eigensolver) adding the error pass to it
// stalled the join (13.9 vs 12.7 ms per solve).
static bool tail_deferred_r(const rtcur_engine* e) {   // (for an RTCUR-R solve)
  static const int defer_env = [] { const char* v = getenv("RTCUR_TAIL_DEFER"); return v ? atoi(v) : -1; }();
  return defer_env >= 0 ? defer_env != 0 : e->P.g.nblk_total * e->P.esize <= ((i64)48 << 20);
}
static bool tail_deferred(const rtcur_engine* e) {
  static const int defer_env = [] { const char* v = getenv("RTCUR_TAIL_DEFER"); return v ? atoi(v) : -1; }();
  return !e->r_mode ? defer_env != 0 : tail_deferred_r(e);
}

// Issue the staging work of a prefetched sample on the side stream (see use_side)
struct SideScope {
  rtcur_engine* e;
  cudaStream_t saved;
  explicit SideScope(rtcur_engine* en) : e(en), saved(en->st) {
    if (e->staging_on_side) e->st = e->side;
  }
  ~SideScope() {
    if (e->staging_on_side) {
      cudaEventRecord(e->side_ev, e->side);
      e->st = saved;
    }
  }
};

extern "C" int rtcur_engine_set_sample(rtcur_engine* e, const int64_t* const* rows, const int64_t* const* cols) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  if (e->npending > 0 && e->use_side && !e->shard && !e->staging_on_side && e->use_graphs) {
    e->staging_on_side = true;
    // eig_ev is recorded inside the running iteration (after pre_ev): waiting for it
    // also covers every earlier reader of the slot being refilled.  With a held-back tail
    // the eigensolver's window already takes the previous iteration's error pass (config 1:
    // 44 us of tail against a 49 us warm eigensolver; adding the 27 us of staging stalled
    // the join by ~20 us): the staging then starts with the SVD post, whose Rayleigh-Ritz
    // tail runs on one CTA per mode
    static const bool late = [] { const char* v = getenv("RTCUR_STAGE_LATE"); return !(v && v[0] == '0'); }();
    CK(cudaStreamWaitEvent(e->side, (late && e->npending > 0 && tail_deferred_r(e)) ? e->svd_ev : e->eig_ev, 0));
  }
  if (e->npending > 0 || e->cur >= 0) e->r_mode = true;   // a sample staged between iterations: RTCUR-R
  SideScope side_scope(e);
  const Plan& P = e->P;
  const Geom& g = P.g;
  const i64 total = [&] { i64 t = 1; for (int m = 0; m < g.n; ++m) t *= g.dim[m]; return t; }();
  // the next sample goes to the inactive slot (stream-ordered after the running
  // iteration, which keeps reading the active one); its pinned index staging is
  // free once that slot's previous upload has completed
  // the slot: the staged one again, else one that is neither the active sample nor (while a
  // speculative iteration may be cancelled) the sample the solve would fall back to
  int slot = e->stg;
  if (slot < 0) {
    slot = 0;
    while (slot == e->act || (e->snap_valid && slot == e->snap.act)) ++slot;
  }
  CK(cudaEventSynchronize(e->idx_ev[slot]));
  i64* h_idx = e->h_idx + (size_t)slot * (e->h_idx_len + 8);
  const i64 sdl = e->sd(slot);
  // validate (fiber_cur.py:67-83) and stage 0-based copies in pinned memory
  // the staging mirrors the slot's device layout (rows_0..rows_n-1, cols_0..cols_n-1
  // as carved by make_plan): one H2D copy of the whole index range
  char* hb = reinterpret_cast<char*>(h_idx);
  for (int m = 0; m < g.n; ++m) {
    int* dst = reinterpret_cast<int*>(hb + (P.o_rows[m] - P.o_rows[0]));
    for (i64 i = 0; i < g.nrows[m]; ++i) {
      const int64_t v = rows[m][i];
      if (v < 1 || v > g.dim[m]) return fail(RT_ERR_INDEX, "mode " + std::to_string(m + 1) + ": row index outside [1, d]");
      if (i > 0 && v <= rows[m][i - 1]) return fail(RT_ERR_VALUE, "row sets must be sorted and unique");
      dst[i] = (int)(v - 1);
    }
  }
  for (int m = 0; m < g.n; ++m) {
    i64* dst = reinterpret_cast<i64*>(hb + (P.o_cols[m] - P.o_rows[0]));
    const i64 rest = total / g.dim[m];
    for (i64 i = 0; i < g.ncols[m]; ++i) {
      const int64_t v = cols[m][i];
      if (v < 1 || v > rest) return fail(RT_ERR_INDEX, "mode " + std::to_string(m + 1) + ": fiber column outside range");
      if (i > 0 && v <= cols[m][i - 1]) return fail(RT_ERR_VALUE, "column sets must be sorted and unique");
      dst[i] = v - 1;
    }
  }
  const i64 span = P.o_cols[g.n - 1] + g.ncols[g.n - 1] * 8 - P.o_rows[0];
  CK(cudaMemcpyAsync(e->ws + P.o_rows[0] + sdl, hb, span, cudaMemcpyHostToDevice, e->st));
  CK(cudaEventRecord(e->idx_ev[slot], e->st));
  IndexPtrs ip = make_ip_slot(e, slot);
  prof_begin(e, PH_PREP);
  dim3 gp((unsigned)std::min<i64>(cdiv(std::max(P.dmax, P.qmax), 256), 4096), g.n + g.nblk);
  k_prep<<<gp, 256, 0, e->st>>>(g, ip, e->at<int>(P.o_rowpos + sdl), e->at<i64>(P.o_colR + sdl),
                                e->at<int>(P.o_coli1 + sdl), e->at<i64>(P.o_coloff));
  LAUNCH_CHECK();
  prof_end(e, PH_PREP);
  e->sampled = true;
  e->stg = slot;
  e->xi_valid[slot] = false;
  return RT_OK;
}

// byte offset (in the workspace) of the compact blocks the next gather writes / the
// next iteration reads: the staged sample slot if any, else the active one
extern "C" int rtcur_engine_xblocks_offset(rtcur_engine* e, int64_t* offset) {
  if (!e || !offset) return fail(RT_ERR_VALUE, "null argument");
  const int slot = e->stg >= 0 ? e->stg : e->act_slot();
  *offset = e->P.o_xb + e->sd(slot);
  e->xi_valid[slot] = false;   // the caller writes the blocks: the intersection copies are refreshed before use
  return RT_OK;
}

static int refresh_xi(rtcur_engine* e, int slot);
static int run_wcols(rtcur_engine* e, double* sto, int sample_slot);
static int alloc_slot(rtcur_engine* e);

// Shadow of the running iteration for the sample just staged on the side stream: a copy of
// its G and A (complete at st_ev, else at the end of its main part) with W evaluated on
// that sample.  The next iteration thresholds against it (reference solver.py:330-331,
// _eval_blocks(lcur, idx) on the new draw) without touching the running iterate's own W,
// which its error pass and the exports still read -- and the evaluation leaves the
// iteration's critical path.
static int make_shadow(rtcur_engine* e, int sample_slot) {
  const Plan& P = e->P;
  e->shadow = -1;
  const int sh = alloc_slot(e);
  if (sh < 0) return RT_OK;   // (no free slot: the next iteration re-evaluates in place)
  CK(cudaStreamWaitEvent(e->st, e->st_ev_seq == e->cur_of_seq ? e->st_ev : e->main_ev, 0));
  CK(cudaMemcpyAsync(e->state(sh), e->state(e->cur), (size_t)P.g.blk[0].w_off * 8, cudaMemcpyDeviceToDevice, e->st));
  e->wt_alt = true;
  const int st = run_wcols(e, e->state(sh), sample_slot);
  e->wt_alt = false;
  if (st) return st;
  e->shadow = sh;
  e->shadow_of = e->cur;
  e->shadow_epoch = e->sample_epoch + 1;
  e->w_epoch[sh] = e->sample_epoch + 1;
  return RT_OK;
}

extern "C" int rtcur_engine_gather(rtcur_engine* e) {
  if (!e || !e->X) return fail(RT_ERR_VALUE, "no tensor bound");
  if (!e->sampled) return fail(RT_ERR_VALUE, "no sample set");
  SideScope side_scope(e);
  const Plan& P = e->P;
  const int slot = e->stg >= 0 ? e->stg : e->act_slot();
  IndexPtrs ip = make_ip_slot(e, slot);
  prof_begin(e, PH_GATHER);
  const bool whole = e->lo == 0 && e->hi == P.g.dim[0];
  // mode copies still being built on the side stream: a gather staged there comes after them
  // in stream order; on the solve's own stream the first gather of a solve reads strided
  // fibers instead of waiting, a later one waits once
  bool copies_ok = true;
  if (e->mcopy_fresh && !e->staging_on_side) {
    if (e->cur < 0 && e->npending == 0) {
      copies_ok = false;
    } else {
      CK(cudaStreamWaitEvent(e->st, e->mcopy_ev, 0));
      e->mcopy_fresh = false;
    }
  }
  ModeCopies mc;
  for (int m = 0; m < RT_MAX_MODES; ++m) mc.p[m] = (whole && copies_ok) ? e->mcopy[m] : nullptr;
  // contiguous fibers (mode 1 of an unsharded X, modes with a mode-k copy): warp-per-column
  // copies that also fill the intersection copies; the rest through the tile gather
  FastGather fg;
  memset(&fg, 0, sizeof(fg));
  TileMap tg = P.tm;
  {
    i64 t = 0;
    for (int b = 0; b < P.g.nblk; ++b) {
      const BlockDesc& bd = P.g.blk[b];
      // large cores: k_gather_core (CW columns per warp); small ones ride along in k_gather_fibers
      const bool core_fast = whole && bd.is_core && bd.P <= 256 && bd.Q >= 100000;
      const bool fast = whole && !core_fast && (bd.is_core || bd.mode == 0 || mc.p[bd.mode] != nullptr);
      if (core_fast) {
        tg.first[b] = t;
        continue;
      }
      const i64 nt = P.tm.first[b + 1] - P.tm.first[b];
      tg.first[b] = t;
      if (fast) {
        fg.blk[fg.nb] = b;
        fg.colbase[fg.nb + 1] = fg.colbase[fg.nb] + bd.Q;
        ++fg.nb;
        fg.src[bd.mode] = (bd.is_core || bd.mode == 0) ? e->X : mc.p[bd.mode];
        if (P.fiber_mask >> b & 1) fg.ximask |= 1u << b;
      } else {
        t += nt;
      }
    }
    tg.first[P.g.nblk] = t;
  }
  fg.xi = e->ws + P.o_xi + e->sd(slot);
  for (int m = 0; m < P.g.n; ++m) {
    fg.xi_off[m] = P.xi_off[m];
    fg.xi_ld[m] = P.xi_ld[m];
  }
  if (tg.first[P.g.nblk] > 0) {
    k_gather<<<(unsigned)tg.first[P.g.nblk], 256, 0, e->st>>>(P.g, tg, ip, e->X, P.dtype, e->lo, e->hi, e->xb(slot), mc);
    LAUNCH_CHECK();
  }
  if (whole && P.g.blk[0].P <= 256 && P.g.blk[0].Q >= 100000) {
    const i64 nw = cdiv(P.g.blk[0].Q, GC_CW);
    const unsigned grid = (unsigned)std::min<i64>(cdiv(nw, 8), 148 * 8);
    const size_t sm = (size_t)P.g.blk[0].P * 4;
    if (P.dtype == 0) k_gather_core<double><<<grid, 256, sm, e->st>>>(P.g, ip, e->X, e->xb(slot));
    else k_gather_core<float><<<grid, 256, sm, e->st>>>(P.g, ip, e->X, e->xb(slot));
    LAUNCH_CHECK();
  }
  if (fg.nb > 0) {
    const unsigned grid = (unsigned)std::min<i64>(cdiv(fg.colbase[fg.nb], 8), 148 * 16);
    if (P.dtype == 0) k_gather_fibers<double><<<grid, 256, 0, e->st>>>(P.g, ip, fg, e->xb(slot));
    else k_gather_fibers<float><<<grid, 256, 0, e->st>>>(P.g, ip, fg, e->xb(slot));
    LAUNCH_CHECK();
  }
  // the intersection copies are complete when every fiber-pass block was copied here
  e->xi_valid[slot] = ((P.fiber_mask & ~1u) & ~fg.ximask) == 0;   // (bit 0: the core, no copy)
  if (int st = refresh_xi(e, slot)) return st;
  prof_end(e, PH_GATHER);
  // staged on the side stream behind a running iteration: evaluate that iterate on this sample too
  static const bool shadow_on = [] { const char* v = getenv("RTCUR_SHADOW"); return !(v && v[0] == '0'); }();
  if (shadow_on && e->staging_on_side && e->npending > 0 && e->cur >= 0 && e->stg == slot && e->use_graphs)
    if (int st = make_shadow(e, slot)) return st;
  return RT_OK;
}

// persistent grid: as many CTAs per SM as the kernel's registers and shared memory allow (<= 4)
template <typename K>
static int launch_bp(K kern, i64 ntiles, i64 smb, cudaStream_t st, const Geom& g, const TileMap& tm,
                     const IndexPtrs& ip, const PassArgs& a, const BPGeom& G) {
  int per_sm = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, (size_t)smb));
  per_sm = std::max(1, std::min(per_sm, 4));
  const unsigned grid = (unsigned)std::max<i64>(1, std::min<i64>(148 * per_sm, ntiles));
  kern<<<grid, 256, smb, st>>>(g, tm, ip, a, G);
  LAUNCH_CHECK();
  return RT_OK;
}

// A pass: fixed grid (the partial-slot layout depends on it)
template <typename K>
static int launch_ap(K kern, int grid, int threads, i64 smb, cudaStream_t st, const Geom& g, const TileMap& tm,
                     const IndexPtrs& ip, const PassArgs& a, const BPGeom& G) {
  kern<<<grid, threads, smb, st>>>(g, tm, ip, a, G);
  LAUNCH_CHECK();
  return RT_OK;
}

// fiber-pass launch description for a sample slot (k_fiber.cuh)
static FiberLaunch make_fl(const rtcur_engine* e, int slot) {
  const Plan& P = e->P;
  FiberLaunch fl;
  memset(&fl, 0, sizeof(fl));
  fl.g = P.g;
  fl.xb = e->xb(slot);
  fl.dtype = P.dtype;
  fl.xi = e->ws + P.o_xi + e->sd(slot);
  const IndexPtrs ip = make_ip_slot(e, slot);
  for (int m = 0; m < P.g.n; ++m) {
    fl.xi_off[m] = P.xi_off[m];
    fl.xi_ld[m] = P.xi_ld[m];
    fl.rows[m] = ip.rows[m];
    fl.rowpos[m] = ip.rowpos[m];
  }
  return fl;
}

// intersection copies of a sample slot, refreshed when its blocks changed
static int refresh_xi(rtcur_engine* e, int slot) {
  if (!e->P.fiber_mask || e->xi_valid[slot]) return RT_OK;
  const int st = fiber_xi_extract(make_fl(e, slot), e->st);
  if (st < 0) return fail(RT_ERR_CUDA, std::string("k_xi_extract: ") + cudaGetErrorString((cudaError_t)(-st)));
  LAUNCH_CHECK();
  e->xi_valid[slot] = true;
  return RT_OK;
}

static CoreLaunch make_cl(rtcur_engine* e, const double* st_s, double zeta, const double* zetap) {
  const Plan& P = e->P;
  const Geom& g = P.g;
  CoreLaunch cl;
  memset(&cl, 0, sizeof(cl));
  cl.stop = g.stop;
  cl.x = e->xb(e->act_slot()) + g.blk[0].off * P.esize;
  cl.dtype = P.dtype;
  cl.P = (int)g.blk[0].P;
  cl.Q = g.blk[0].Q;
  cl.r = g.rank[0];
  cl.rows0 = make_ip(e).rows[0];
  cl.dA = g.dim[0];
  cl.a_off = g.a_off[0];
  cl.w_off = g.blk[0].w_off;
  cl.st_s = st_s;
  cl.zeta = zeta;
  cl.zetap = zetap;
  return cl;
}

static int run_block_pass(rtcur_engine* e, const double* st_s, const double* st_e, double zeta, bool with_M,
                          double* s_out, double* c_out, double* l_out, bool sums, int phase) {
  const Plan& P = e->P;
  IndexPtrs ip = make_ip(e);
  PassArgs a;
  memset(&a, 0, sizeof(a));
  a.xb = e->xb(e->act_slot());
  a.dtype = P.dtype;
  a.st_s = st_s;
  a.st_e = st_e;
  a.zeta = zeta;
  a.zetap = e->zetap_cur;
  if (with_M)
    for (int m = 0; m < P.g.n; ++m) a.M[m] = e->at<double>(P.o_M[m]);
  a.s_out = s_out;
  a.c_out = c_out;
  a.l_out = l_out;
  if (sums) {
    a.partial = e->at<double>(P.o_bpart);
    a.sums = e->at<double>(P.o_sums + e->roff());
    a.counter = e->at<unsigned int>(P.o_counters);
  }
  a.nonfinite = e->at<int>(P.o_nonfinite + e->roff());
  prof_begin(e, phase);
  const i64 smb = bp_smem_bytes(P.bp);
  const bool hs = st_s != nullptr, he = st_e != nullptr;
  // the fiber blocks of the threshold / error passes go to the TMA fiber pass; exports stay here
  const bool split = !(s_out || c_out || l_out) && ((with_M && !sums && P.fb_thr) || (sums && (P.fb_err || P.core_k)));
  const bool thr_only = with_M && !sums && !(s_out || c_out || l_out);
  const TileMap& tmk = thr_only ? P.tm_thr : split ? P.tm_core : P.tm;
#define BP_LAUNCH(HS, HE, WM, EXP)                                                                        \
  (P.rb == 4    ? launch_bp(k_block_pass<HS, HE, WM, EXP, false, 4, false>, tmk.first[P.g.nblk], smb, e->st, P.g, tmk,  \
                            ip, a, P.bp)                                                                          \
   : P.rb == 8  ? launch_bp(k_block_pass<HS, HE, WM, EXP, false, 8, false>, tmk.first[P.g.nblk], smb, e->st, P.g, tmk,  \
                            ip, a, P.bp)                                                                          \
   : P.rb == 16 ? launch_bp(k_block_pass<HS, HE, WM, EXP, false, 16, false>, tmk.first[P.g.nblk], smb, e->st, P.g,      \
                            tmk, ip, a, P.bp)                                                                    \
                : launch_bp(k_block_pass<HS, HE, WM, EXP, false, 32, false>, tmk.first[P.g.nblk], smb, e->st, P.g,      \
                            tmk, ip, a, P.bp))
  int lst = 0;
  if (tmk.first[P.g.nblk] == 0) {
    // nothing left for k_block_pass (threshold pass with every fiber block on the fiber pass)
  } else if (s_out || c_out || l_out) {
    if (hs && he) lst = BP_LAUNCH(true, true, false, true);
    else if (hs) lst = BP_LAUNCH(true, false, false, true);
    else if (he) lst = BP_LAUNCH(false, true, false, true);
    else lst = BP_LAUNCH(false, false, false, true);
  } else if (with_M) {
    if (hs) lst = BP_LAUNCH(true, false, true, false);
    else lst = BP_LAUNCH(false, false, true, false);
  } else {
    if (hs) lst = BP_LAUNCH(true, true, false, false);
    else lst = BP_LAUNCH(false, true, false, false);
  }
#undef BP_LAUNCH
  if (lst) return lst;
  if (split && sums && P.core_k) {
    // the core's share of the error pass (sums of block 0)
    CoreLaunch cl = make_cl(e, st_s, zeta, a.zetap);
    cl.mode = 1;
    cl.st_e = st_e;
    cl.partial = e->at<double>(P.o_cpart);
    cl.sums = a.sums;
    cl.counter = e->at<unsigned int>(P.o_counters) + 48;
    const int cst = core_pass_launch(cl, e->st);
    if (cst < 0) return fail(RT_ERR_CUDA, std::string("k_core_pass (error): ") + cudaGetErrorString((cudaError_t)(-cst)));
    rtcur_launch_counter_add(1);
  }
  if (split && (sums ? P.fb_err : P.fb_thr)) {
    FiberLaunch fl = make_fl(e, e->act_slot());
    fl.mask = sums ? P.fb_err : P.fb_thr;
    fl.st_s = st_s;
    fl.st_e = st_e;
    fl.zeta = zeta;
    fl.zetap = a.zetap;
    for (int m = 0; m < P.g.n; ++m) fl.M[m] = a.M[m];
    fl.reserve_sms = sums ? e->tail_reserve : 0;
    fl.partial = a.partial;
    fl.sums = a.sums;
    fl.counter = a.counter;
    fl.nonfinite = a.nonfinite;
    const int fst = fiber_pass_launch(fl, e->st);
    if (fst < 0) return fail(RT_ERR_CUDA, std::string("k_fiber_pass: ") + cudaGetErrorString((cudaError_t)(-fst)));
    rtcur_launch_counter_add((unsigned long long)fst);
  }
  prof_end(e, phase);
  return RT_OK;
}

static SvdArgs make_svd_args(rtcur_engine* e) {
  const Plan& P = e->P;
  SvdArgs sa;
  memset(&sa, 0, sizeof(sa));
  sa.stop = P.g.stop;
  sa.n = P.g.n;
  for (int m = 0; m < P.g.n; ++m) {
    sa.s[m] = (int)P.s[m];
    sa.l[m] = P.l[m];
    sa.r[m] = P.g.rank[m];
    sa.tall[m] = P.tall[m];
    sa.mrows[m] = P.g.nrows[m];
    sa.pcols[m] = P.g.ncols[m];
    sa.M[m] = e->at<double>(P.o_M[m]);
    sa.E[m] = e->at<double>(P.o_E[m]);
    sa.Z[m] = e->at<double>(P.o_Z[m]);
    sa.hpart[m] = e->at<double>(P.o_hpart[m]);
    sa.H[m] = e->at<double>(P.o_H[m]);
    sa.Q[m] = e->at<double>(P.o_Q[m]);
    sa.U[m] = e->at<double>(P.o_U[m]);
    sa.V[m] = e->at<double>(P.o_V[m]);
    sa.sig[m] = e->at<double>(P.o_sig[m]);
    sa.siginv[m] = e->at<double>(P.o_siginv[m]);
    sa.perm[m] = e->at<int>(P.o_perm[m]);
    sa.degen[m] = e->at<int>(P.o_degen[m]);
  }
  sa.flags = e->at<int>(P.o_flags + e->roff());
  sa.hchunk = P.hchunk;
  return sa;
}

// rank-r truncated SVD of every mode's intersection M_k (already in the workspace)
// k_eig: one CTA per mode, or clusters of EIG_CLUSTER CTAs per mode when some
// intersection has 128 < s <= 256 (their tridiagonalisation is spread over the
// cluster's registers, k_eig.cu eig_tridiag_reg)
static int launch_eig(const EigArgs& ea, const i64* s, int n, int esm, cudaStream_t st) {
  bool clus = false;
  for (int m = 0; m < n; ++m) clus |= ea.reg_tridiag && s[m] > 128 && s[m] <= 256;
  if (!clus) {
    k_eig<<<n, EIG_THREADS, esm, st>>>(ea);
    LAUNCH_CHECK();
    return RT_OK;
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)(n * EIG_CLUSTER));
  cfg.blockDim = dim3(EIG_THREADS);
  cfg.dynamicSmemBytes = (size_t)esm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = EIG_CLUSTER;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_eig, ea));
  LAUNCH_CHECK();
  return RT_OK;
}

static int run_svd(rtcur_engine* e, const double* warm_state) {
  const Plan& P = e->P;
  const int n = P.g.n;
  static const bool kfull_on = [] { const char* v = getenv("RTCUR_EIG_KFULL"); return !(v && v[0] == '0'); }();
  GramArgs ga;
  memset(&ga, 0, sizeof(ga));
  ga.stop = P.g.stop;
  ga.n = n;
  for (int m = 0; m < n; ++m) {
    ga.s[m] = (int)P.s[m];
    ga.l[m] = P.l[m];
    ga.tall[m] = P.tall[m];
    ga.mrows[m] = P.g.nrows[m];
    ga.M[m] = e->at<double>(P.o_M[m]);
    ga.K[m] = e->at<double>(P.o_K[m]);
    ga.Kfull[m] = (kfull_on && P.s[m] > 128) ? e->at<double>(P.o_Kfull[m]) : nullptr;
  }
  ga.part = e->at<double>(P.o_gpart);
  ga.maxchunks = P.gram_maxchunks;
  ga.maxpairs = P.gram_maxpairs;
  ga.cl = P.gram_cl;
  prof_begin(e, PH_GRAM);
  {
    // fp64 tensor cores (DMMA) unless RTCUR_GRAM_DMMA=0
    static const bool dmma = [] { const char* v = getenv("RTCUR_GRAM_DMMA"); return !(v && v[0] == '0'); }();
    if (dmma) k_gram_tiles_dmma<<<dim3(P.gram_maxpairs, P.gram_maxchunks, n), 128, 0, e->st>>>(ga);
    else k_gram_tiles<<<dim3(P.gram_maxpairs, P.gram_maxchunks, n), 256, 0, e->st>>>(ga);
  }
  LAUNCH_CHECK();
  {
    const i64 npk = P.smax * (P.smax + 1) / 2;
    k_gram_reduce<<<dim3((unsigned)std::min<i64>(cdiv(npk * 32, 256), 2048), n), 256, 0, e->st>>>(ga);
    LAUNCH_CHECK();
  }
  prof_end(e, PH_GRAM);
  EigArgs ea;
  memset(&ea, 0, sizeof(ea));
  ea.stop = P.g.stop;
  ea.n = n;
  int esm = 0;
  for (int m = 0; m < n; ++m) {
    ea.s[m] = (int)P.s[m];
    ea.r[m] = P.g.rank[m];
    ea.K[m] = e->at<double>(P.o_K[m]);
    ea.Kfull[m] = ga.Kfull[m];
    ea.E[m] = e->at<double>(P.o_E[m]);
    ea.lam[m] = e->at<double>(P.o_lam[m]);
    ea.nb[m] = P.nb[m];
    ea.lug[m] = P.lug[m] ? e->at<double>(P.o_lug[m]) : nullptr;
    ea.full[m] = eig_pick_full((int)P.s[m], P.g.rank[m]);
    esm = std::max(esm, eig_smem_bytes(P, m));
  }
  // Lanczos full path: the Krylov basis goes after the mode's base layout
  {
    static const bool lz = [] { const char* v = getenv("RTCUR_EIG_LANCZOS"); return !(v && v[0] == '0'); }();
    for (int m = 0; m < n; ++m) {
      const int sm = (int)P.s[m], rm = P.g.rank[m];
      const long long base = eig_smem_doubles(sm, rm, P.nb[m], ea.full[m], eig_fast_ok(P, m));
      const int mcap = lz ? eig_lz_mcap(sm, rm, base, ea.full[m]) : 0;
      ea.lz_mcap[m] = mcap;
      ea.lz_off[m] = (int)base;
      if (mcap && ea.full[m]) esm = std::max(esm, (int)((base + (long long)sm * (mcap + 1) + 2 * (mcap + 1) + 8) * 8));
    }
  }
  {
    static const int lzs = [] { const char* v = getenv("RTCUR_LZ_STRIDE"); return v ? std::max(1, atoi(v)) : 8; }();
    ea.lz_stride = lzs;
  }
  ea.tmark = e->at<long long>(P.o_dbg);
  // certified attempts take <= 15 steps at configs 0-4 (tools/eig_paths.py); a
  // failing one is capped near the full path's cost
  ea.max_sub_steps = 16;
  {
    static const int msw = [] { const char* v = getenv("RTCUR_EIG_MS_WARPS"); return v ? std::max(1, atoi(v)) : 1; }();
    ea.ms_warps = msw;
  }
  ea.fast_used = e->at<int>(P.o_fast);
  {
    // register-tiled tridiagonalisation: 1 (default) for 128 < s <= 256 (cluster of
    // EIG_CLUSTER CTAs; 1.3-1.6x on that phase), 2 also single-CTA for s <= 128
    // (measured no faster than the shared-memory path there), 0 off
    static const int reg = [] { const char* v = getenv("RTCUR_EIG_REG"); return v ? atoi(v) : 1; }();
    ea.reg_tridiag = reg;
  }
  IndexPtrs ipw = make_ip(e);
  for (int m = 0; m < n; ++m) {
    // fast path only for wide intersections (short side = rows I_k) with a previous iterate
    ea.warmA[m] = (warm_state && eig_fast_ok(P, m) && e->use_fast) ? warm_state + P.g.a_off[m] : nullptr;
    ea.warm_rows[m] = ipw.rows[m];
    ea.warm_d[m] = P.g.dim[m];
  }
  // the next sample's prefetch (side stream) may start now: it overlaps the eigensolver
  if (e->capturing) cap_cut(e, CUT_EIG, 0);
  else CK(cudaEventRecord(e->eig_ev, e->st));
  prof_begin(e, PH_EIG);
  if (int st = launch_eig(ea, P.s, n, esm, e->st)) return st;
  prof_end(e, PH_EIG);
  // the previous iteration's tail (enqueued under this eigensolver) sets the stop flag:
  // everything from here on must see it
  if (e->capturing) cap_cut(e, CUT_JOIN, 0);
  prof_begin(e, PH_SVDPOST);
  SvdArgs sa = make_svd_args(e);
  unsigned int* hcnt = e->at<unsigned int>(P.o_counters) + 16;
  const unsigned gz = (unsigned)cdiv(P.lmax, 256);
  const int zsm = (int)(P.smax * (P.rmax + ZP_LD) * 8);
  DISPATCH_R(P.rb, k_zproj, dim3((unsigned)cdiv(P.lmax, ZP_T), n), 32 * P.rb, zsm, e->st, sa);
  LAUNCH_CHECK();
  const int hsm = (int)((std::max<i64>(HG_CH * P.rmax + 512, 7 * P.rmax * P.rmax + 3 * P.rmax + 8)) * 8);
  // H = Z^T Z -> (last CTA) Rayleigh-Ritz rotation, short-side vectors, then sigma,
  // order, cutoff, flags and T' from H' = Q^T H Q
  k_hgram<3><<<dim3(P.h_maxchunks, n), 512, hsm, e->st>>>(sa, hcnt);
  LAUNCH_CHECK();
  // long side Z T -> (last CTA) short-side permutation + completion
  DISPATCH_R(P.rb, k_long, dim3(gz, n), 256, 0, e->st, sa, hcnt + 8);
  LAUNCH_CHECK();
  prof_end(e, PH_SVDPOST);
  return RT_OK;
}

// Expanding chain out = G x_2 B_2 x_3 .. x_n B_n with B_m = A_m(rows_m, :) (rows_m null:
// all d_m rows), written to `dst` in (r1, P_2, .., P_n) F-order.
static int run_wchain(rtcur_engine* e, const double* sto, const int* const* rows, const i64* Pm, double* dst) {
  const Plan& P = e->P;
  const Geom& g = P.g;
  const int n = g.n;
  if (n == 1) {
    CK(cudaMemcpyAsync(dst, sto, g.gsize * 8, cudaMemcpyDeviceToDevice, e->st));
    return RT_OK;
  }
  double* t0 = e->at<double>(e->wt_alt ? P.o_wt0s : P.o_wt0);
  double* t1 = e->at<double>(e->wt_alt ? P.o_wt1s : P.o_wt1);
  const double* in = sto;   // G
  i64 rho = g.rank[0];
  for (int m = 1; m < n; ++m) {
    i64 beta = 1;
    for (int l = m + 1; l < n; ++l) beta *= g.rank[l];
    double* out = (m == n - 1) ? dst : (in == t0 ? t1 : t0);
    const i64 total = rho * Pm[m] * beta;
    k_modeprod_fwd<<<(unsigned)std::min<i64>(cdiv(total, 256), 148 * 16), 256, 0, e->st>>>(
        in, out, sto + g.a_off[m], rows ? rows[m] : nullptr, g.dim[m], rho, Pm[m], g.rank[m], beta, g.stop);
    LAUNCH_CHECK();
    rho *= Pm[m];
    in = out;
  }
  return RT_OK;
}

// W_b of every block column for state `sto`: the core by the separable chain,
// the fiber blocks (arbitrary multi-indices) by k_wcols
static int run_wcols(rtcur_engine* e, double* sto, int sample_slot) {
  const Plan& P = e->P;
  const Geom& g = P.g;
  IndexPtrs ip = make_ip_slot(e, sample_slot);
  prof_begin(e, PH_WCOLS);
  // large cores: separable chain (r_m FMAs per output); small ones stay in the
  // single k_wcols launch (launch overhead dominates there)
  const bool chain = g.n >= 2 && g.blk[0].Q * (g.gsize / g.rank[0]) > (i64)2000000;
  // the core's chain and the fiber blocks' kernel are independent: two branches of the graph
  // in a captured iteration (RTCUR_W_FORK=0: in order)
  static const bool w_fork = [] { const char* v = getenv("RTCUR_W_FORK"); return !(v && v[0] == '0'); }();
  const bool forked = chain && w_fork && e->capturing && e->cap_st2 != nullptr && e->st != e->cap_st2;
  cudaStream_t st_main = e->st;
  if (chain) {
    const int* rows[RT_MAX_MODES];
    i64 Pm[RT_MAX_MODES];
    for (int m = 0; m < g.n; ++m) { rows[m] = ip.rows[m]; Pm[m] = g.nrows[m]; }
    if (forked) {
      CK(cudaEventRecord(e->fork_ev, st_main));
      CK(cudaStreamWaitEvent(e->cap_st2, e->fork_ev, 0));
      e->st = e->cap_st2;
    }
    int st = run_wchain(e, sto, rows, Pm, sto + g.blk[0].w_off);
    e->st = st_main;
    if (st) return st;
  }
  i64 qf = 1;
  for (int b = chain ? 1 : 0; b < g.nblk; ++b) qf = std::max(qf, g.blk[b].Q);
  // warp per column with the rank combinations over the lanes when its tables fit
  i64 ncmax = 1, rsmax = 1;
  for (int t = 0; t < g.n; ++t) {
    i64 nc = 1, rs = 0;
    for (int m = 0; m < g.n; ++m)
      if (m != t) { nc *= g.rank[m]; rs += g.rank[m]; }
    ncmax = std::max(ncmax, nc);
    rsmax = std::max(rsmax, rs);
  }
  // lanes per column: a warp for many combinations, 8 lanes (4 columns per warp) for a few
  static const int gs_env = [] { const char* v = getenv("RTCUR_WC_GS"); return v ? atoi(v) : 0; }();
  // (8 lanes also when each column has many outputs: the per-output shuffle trees
  // dominate; measured: configs 2/3 wcols -21/-27 %, config 4 (r = 4) better on 32)
  const int gs = (gs_env == 8 || gs_env == 32) ? gs_env : ((ncmax >= 48 && P.rb < 8) ? 32 : 8);
  const int ngrp = 32 * WC_WARPS / gs;
  const int rows_cap = (int)(cdiv(rsmax, gs) * gs);
  const i64 wsm = (g.gsize + (ncmax * 4 + ncmax * std::max(1, g.n - 1) + 7) / 8 + 1 + (i64)ngrp * rows_cap) * 8;
  if (wsm <= 200 * 1024 && ncmax >= 8) {   // very few combinations: a thread per column is cheaper
    // columns per lane group and pass (RTCUR_WC_CPG; 1: +0.4..1.8 % over 2 at configs 0-4)
    static const int cpg = [] { const char* v = getenv("RTCUR_WC_CPG"); return v ? std::max(1, atoi(v)) : 1; }();
    const dim3 grid((unsigned)std::min<i64>(cdiv(qf, ngrp * cpg), 148 * 4 * (cpg == 1 ? 2 : 1)), g.nblk);
#define WCW(RB, GS) k_wcols_warp<RB, GS><<<grid, 32 * WC_WARPS, (int)wsm, e->st>>>(g, ip, sto, chain ? 1 : 0, rows_cap)
    if (gs == 32) {
      switch (P.rb) {
        case 4: WCW(4, 32); break;
        case 8: WCW(8, 32); break;
        case 16: WCW(16, 32); break;
        default: WCW(32, 32); break;
      }
    } else {
      switch (P.rb) {
        case 4: WCW(4, 8); break;
        case 8: WCW(8, 8); break;
        case 16: WCW(16, 8); break;
        default: WCW(32, 8); break;
      }
    }
#undef WCW
  } else {
    const int rpt = wcols_rows_per_thread(g);
    DISPATCH_R(P.rb, k_wcols, dim3((unsigned)cdiv(qf, 128), g.nblk), 128, wcols_smem(g), e->st, g, ip, sto, 0,
               (double*)nullptr, rpt, chain ? 1 : 0);
  }
  LAUNCH_CHECK();
  if (forked) {   // join the core chain's branch
    CK(cudaEventRecord(e->join2_ev, e->cap_st2));
    CK(cudaStreamWaitEvent(st_main, e->join2_ev, 0));
  }
  prof_end(e, PH_WCOLS);
  return RT_OK;
}

// A_k, G, W of the new iterate into state slot `dst` (threshold from st_s)
static int run_factors(rtcur_engine* e, const double* st_s, double zeta, int dst) {
  const Plan& P = e->P;
  const Geom& g = P.g;
  const int n = g.n;
  IndexPtrs ip = make_ip(e);
  double* sto = e->state(dst);
  // The A pass (fiber blocks -> A_k) and the G pass (core -> G) are independent: in a
  // captured iteration they are two branches of the graph (fork here, join before the
  // column weights), so their launch ramps and reduction tails overlap
  // (RTCUR_AG_FORK=0: one after the other).
  static const bool ag_fork = [] { const char* v = getenv("RTCUR_AG_FORK"); return !(v && v[0] == '0'); }();
  const bool forked = ag_fork && e->capturing && e->cap_st2 != nullptr;
  cudaStream_t st_main = e->st;
  if (forked) {
    CK(cudaEventRecord(e->fork_ev, st_main));
    CK(cudaStreamWaitEvent(e->cap_st2, e->fork_ev, 0));
  }
  prof_begin(e, PH_APASS);
  // A_k = C_k V_k S_k^+: the fiber pass for its blocks (all of them in the usual case),
  // the block-pass A pass when some fiber block is outside its envelope
  unsigned all_fibers = 0;
  for (int b = 1; b < g.nblk; ++b) all_fibers |= 1u << b;
  if ((P.fb_ap & all_fibers) != all_fibers) {
    const TileMap& tma = P.tm_ap;   // the fiber blocks the fiber pass does not take
    // A_k = C_k V_k S_k^+ on the block-pass tiles (fiber blocks), then the fixed-order reduction
    PassArgs pa;
    memset(&pa, 0, sizeof(pa));
    pa.xb = e->xb(e->act_slot());
    pa.dtype = P.dtype;
    pa.st_s = st_s;
    pa.zeta = zeta;
    pa.zetap = e->zetap_cur;
    for (int m = 0; m < n; ++m) {
      pa.V[m] = e->at<double>(P.o_V[m]);
      pa.siginv[m] = e->at<double>(P.o_siginv[m]);
    }
    pa.apart = e->at<double>(P.o_apart2);
    // never more CTAs than the map's fiber tiles: a CTA with an empty tile range would
    // leave its partial slot unwritten while the reduction reads it
    const int apg = (int)std::max<i64>(1, std::min<i64>(P.ap_grid, tma.first[g.nblk] - tma.first[1]));
    pa.ap_grid = apg;
    pa.nonfinite = e->at<int>(P.o_nonfinite + e->roff());
    const i64 smb = bp_smem_bytes(P.bp_ap);
#define AP_LAUNCH(RB)                                                                                  \
  (st_s ? launch_ap(k_block_pass<true, false, false, false, false, RB, true>, apg, P.ap_threads, smb, e->st, g, tma, ip, pa, \
                    P.bp_ap)                                                                             \
        : launch_ap(k_block_pass<false, false, false, false, false, RB, true>, apg, P.ap_threads, smb, e->st, g, tma, ip, pa, \
                    P.bp_ap))
    int lst;
    switch (P.rb) {
      case 4: lst = AP_LAUNCH(4); break;
      case 8: lst = AP_LAUNCH(8); break;
      case 16: lst = AP_LAUNCH(16); break;
      default: lst = AP_LAUNCH(32); break;
    }
#undef AP_LAUNCH
    if (lst) return lst;
    i64 maxpr = 1;
    for (int b = 1; b < g.nblk; ++b) maxpr = std::max<i64>(maxpr, g.blk[b].P * g.blk[b].r);
    k_areduce_bp<<<dim3((unsigned)std::min<i64>(cdiv(maxpr, 256), 1024), g.nblk - 1), 256, 0, e->st>>>(g, tma, pa, sto);
    LAUNCH_CHECK();
  }
  if (P.fb_ap) {
    FiberLaunch fl = make_fl(e, e->act_slot());
    fl.mask = P.fb_ap;
    fl.st_s = st_s;
    fl.zeta = zeta;
    fl.zetap = e->zetap_cur;
    fl.ap = 1;
    for (int m = 0; m < n; ++m) {
      fl.Vr[m] = e->at<double>(P.o_V[m]);
      fl.siginv[m] = e->at<double>(P.o_siginv[m]);
    }
    fl.apart = e->at<double>(P.o_fapart);
    fl.apart_cap = P.fapart_cap;
    fl.a_out = sto;
    fl.nonfinite = e->at<int>(P.o_nonfinite + e->roff());
    const int fst = fiber_pass_launch(fl, e->st);
    if (fst < 0) return fail(RT_ERR_CUDA, std::string("k_fiber_pass (A): ") + cudaGetErrorString((cudaError_t)(-fst)));
    rtcur_launch_counter_add((unsigned long long)fst);
  }
  prof_end(e, PH_APASS);
  if (forked) e->st = e->cap_st2;   // the G pass's branch
  prof_begin(e, PH_GPASS);
  // G = clean_core x_1 U_1^T x_2 ... x_n U_n^T
  GPassArgs gp;
  memset(&gp, 0, sizeof(gp));
  gp.xb = e->xb(e->act_slot());
  gp.dtype = P.dtype;
  gp.st_s = st_s;
  gp.zeta = zeta;
  gp.zetap = e->zetap_cur;
  for (int m = 0; m < n; ++m) gp.U[m] = e->at<double>(P.o_U[m]);
  double* t0 = e->at<double>(P.o_gt0);
  double* t1 = e->at<double>(P.o_gt1);
  gp.t1 = (n == 1) ? sto : t0;
  {
    // first contraction t1 = clean_core x_1 U~_1^T on the block-pass tiles (lanes over columns)
    IndexPtrs ipg = make_ip(e);
    PassArgs pa;
    memset(&pa, 0, sizeof(pa));
    pa.xb = e->xb(e->act_slot());
    pa.dtype = P.dtype;
    pa.st_s = st_s;
    pa.zeta = zeta;
    pa.zetap = e->zetap_cur;
    pa.U = gp.U[0];
    pa.t1 = gp.t1;
    pa.nonfinite = e->at<int>(P.o_nonfinite + e->roff());
    const BPGeom& G = P.bp_gp;
    const i64 smb = bp_smem_bytes(G);
    if (P.core_k) {
      CoreLaunch cl = make_cl(e, st_s, zeta, e->zetap_cur);
      cl.mode = 0;
      cl.U = gp.U[0];
      cl.t1 = gp.t1;
      const int cst = core_pass_launch(cl, e->st);
      if (cst < 0) return fail(RT_ERR_CUDA, std::string("k_core_pass (G): ") + cudaGetErrorString((cudaError_t)(-cst)));
      rtcur_launch_counter_add(1);
    } else if (P.tm_gp.cols[0]) {
      int lst;
#define GP_LAUNCH(RB)                                                                                      \
  (st_s ? launch_bp(k_block_pass<true, false, false, false, true, RB, false>, P.tm_gp.first[1], smb, e->st, g, P.tm_gp, \
                    ipg, pa, G)                                                                              \
        : launch_bp(k_block_pass<false, false, false, false, true, RB, false>, P.tm_gp.first[1], smb, e->st, g,       \
                    P.tm_gp, ipg, pa, G))
      switch (rbucket(g.rank[0])) {
        case 4: lst = GP_LAUNCH(4); break;
        case 8: lst = GP_LAUNCH(8); break;
        case 16: lst = GP_LAUNCH(16); break;
        default: lst = GP_LAUNCH(32); break;
      }
#undef GP_LAUNCH
      if (lst) return lst;
    } else {   // tall core tiles (fewer than 32 columns fit a stage): warp per column
      const i64 Q = g.blk[0].Q;
      DISPATCH_R(rbucket(g.rank[0]), k_gpass, (unsigned)cdiv(Q * 32, 256), 256, 0, e->st, g, ipg, gp);
      LAUNCH_CHECK();
    }
  }
  {
    i64 rho = g.rank[0];
    const double* in = t0;
    for (int m = 1; m < n; ++m) {
      i64 beta = 1;
      for (int l = m + 1; l < n; ++l) beta *= g.nrows[l];
      double* out = (m == n - 1) ? sto : (in == t0 ? t1 : t0);
      const i64 total = rho * g.rank[m] * beta;
      k_modeprod<<<(unsigned)std::min<i64>(cdiv(total * 32, 256), 4096), 256, 0, e->st>>>(
          in, out, e->at<double>(P.o_U[m]), rho, (int)g.nrows[m], g.rank[m], beta, g.stop);
      LAUNCH_CHECK();
      rho *= g.rank[m];
      in = out;
    }
  }
  prof_end(e, PH_GPASS);
  if (forked) {   // join
    CK(cudaEventRecord(e->join2_ev, e->cap_st2));
    e->st = st_main;
    CK(cudaStreamWaitEvent(st_main, e->join2_ev, 0));
  }
  // G and A of the new iterate are complete: the side stream may evaluate it on the next sample
  if (e->capturing) {
    if (e->r_mode) cap_cut(e, CUT_STATE, 0);
  } else {
    CK(cudaEventRecord(e->st_ev, e->st));
    e->st_ev_seq = e->cur_seq;
  }
  // W for every block column (w_epoch of the new slot is set by the caller).  RTCUR-R: the
  // next iteration evaluates this iterate on ITS sample (shadow or in place), so W on the
  // current sample feeds only the error pass and the exports: it opens the tail instead
  if (e->r_mode) return RT_OK;
  return run_wcols(e, sto, e->act_slot());
}

// Device-side stop rule: the sampled relative error from the per-block sums, in the
// host's own operation order (solver._error_from_sums: sum of block norms over sum of
// block norms, IEEE sqrt / divide), against eps.  Sets the engine's stop flag -- the kernels
// of an iteration enqueued behind this one then return at once -- and its copy in the
// result range the host reads.
static __global__ void k_stop_check(const double* sums, int nblk, const double* ctl, int* stop, int* stop_copy) {
  if (threadIdx.x != 0 || *reinterpret_cast<volatile int*>(stop)) return;   // (a cancelled iteration keeps the flag)
  double num = 0.0, den = 0.0;
  for (int b = 0; b < nblk; ++b) {
    num += sqrt(sums[2 * b]);
    den += sqrt(sums[2 * b + 1]);
  }
  const double err = den == 0.0 ? (num == 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000LL)) : num / den;
  const double eps = ctl[1];
  const int s = (eps > 0.0 && err <= eps) ? 1 : 0;
  *stop = s;
  *stop_copy = s;
}

#define RES_SLOT 96   // doubles between the two result slots in h_pinned (zeta/eps slots at 200 + 4 par)

// The launch sequence of one iteration, in two parts (each captured into CUDA graph
// segments per launch shape).  Pure stream work: host-side bookkeeping stays in the caller.
// Main part: everything the NEXT iteration's threshold depends on.
static int iterate_main(rtcur_engine* e, const double* st_s, int newslot, bool reeval, int par) {
  const Plan& P = e->P;
  const double zeta = e->zeta_last;   // (kernels read the device copy when zetap_cur is set)
  CK(cudaMemcpyAsync(e->ws + P.o_zeta + 32 * par, e->h_pinned + 200 + 4 * par, 16, cudaMemcpyHostToDevice, e->st));
  CK(cudaMemsetAsync(e->ws + P.o_nonfinite + e->roff(), 0, 4, e->st));
  int st;
  // RTCUR-R without a shadow state: the sample moved, re-evaluate the previous iterate on
  // it in place (reference solver.py:330-331, _eval_blocks(lcur, idx) on the new draw)
  if (reeval && (st = run_wcols(e, e->state(e->cur), e->act_slot()))) return st;
  if ((st = refresh_xi(e, e->act_slot()))) return st;
  if ((st = run_block_pass(e, st_s, nullptr, zeta, true, nullptr, nullptr, nullptr, false, PH_THRESH))) return st;
  if ((st = run_svd(e, st_s))) return st;
  return run_factors(e, st_s, zeta, newslot);
}

// Tail: the sampled error of the new iterate, the stop rule, the result copy.
static int iterate_tail(rtcur_engine* e, const double* st_s, int newslot, int par) {
  const Plan& P = e->P;
  int st;
  // a held-back tail runs beside the next eigensolver: one CTA per mode, or a cluster of
  // EIG_CLUSTER per mode when some short side exceeds 128 (see launch_eig)
  e->tail_reserve = 0;
  if (e->capturing && tail_deferred(e)) {
    bool clus = false;
    for (int m = 0; m < P.g.n; ++m) clus |= P.s[m] > 128 && P.s[m] <= 256;
    e->tail_reserve = P.g.n * (clus ? EIG_CLUSTER : 1);
  }
  if (e->r_mode && (st = run_wcols(e, e->state(newslot), e->act_slot()))) return st;   // (see run_factors)
  if ((st = run_block_pass(e, st_s, e->state(newslot), e->zeta_last, false, nullptr, nullptr, nullptr, true, PH_ERROR)))
    return st;
  k_stop_check<<<1, 32, 0, e->st>>>(e->at<double>(P.o_sums + e->roff()), P.g.nblk, e->at<double>(P.o_zeta + 32 * par),
                                    stop_flag(e), e->at<int>(P.o_nonfinite + 4 + e->roff()));
  LAUNCH_CHECK();
  CK(cudaMemcpyAsync(e->h_pinned + par * RES_SLOT, e->ws + P.o_sums + e->roff(), P.res_bytes, cudaMemcpyDeviceToHost,
                     e->st));
  e->tail_reserve = 0;
  return RT_OK;
}

// phases timed inside the iteration body (they cut its graph into segments)
static const unsigned kIterPhases = (1u << PH_THRESH) | (1u << PH_GRAM) | (1u << PH_EIG) | (1u << PH_SVDPOST) |
                                    (1u << PH_APASS) | (1u << PH_GPASS) | (1u << PH_WCOLS) | (1u << PH_ERROR);

static inline bool fiber_refresh_pending(const rtcur_engine* e) {
  return e->P.fiber_mask && !e->xi_valid[e->act_slot()];
}

// capture one iteration into `ge`: the main part's segments, then the tail's
static int capture_iteration(rtcur_engine* e, GraphEntry& ge, const double* st_s, int newslot, bool reeval, int par) {
  e->cap_entry = &ge;
  e->cap_err = (int)cudaSuccess;
  cudaStream_t saved = e->st;
  e->st = e->cap_st;
  e->capturing = true;
  int st = RT_OK;
  cudaError_t ce = cudaSuccess;
  for (int part = 0; part < 2 && st == RT_OK && ce == cudaSuccess; ++part) {
    e->cap_segs = part == 0 ? &ge.segs : &ge.tail;
    const unsigned long long l0 = rtcur_launch_counter_add(0);
    ce = seg_begin(e);
    if (ce != cudaSuccess) break;
    st = part == 0 ? iterate_main(e, st_s, newslot, reeval, par) : iterate_tail(e, st_s, newslot, par);
    const unsigned long long nk = rtcur_launch_counter_add(0) - l0;
    g_launches.fetch_sub(nk);   // capturing executes nothing
    (part == 0 ? ge.nkernels : ge.nk_tail) = nk;
    ce = seg_end(e, CUT_NONE, 0);
    if (ce == cudaSuccess) ce = (cudaError_t)e->cap_err;
  }
  e->capturing = false;
  e->st = saved;
  e->cap_entry = nullptr;
  e->cap_segs = nullptr;
  if (ce != cudaSuccess || st != RT_OK) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(e->cap_st, &junk);   // leave no capture open
    if (junk) cudaGraphDestroy(junk);
    cudaGetLastError();
    for (auto* v : {&ge.segs, &ge.tail}) {
      for (auto& sg : *v)
        if (sg.exec) cudaGraphExecDestroy(sg.exec);
      v->clear();
    }
    if (st) return st;
    return fail(RT_ERR_CUDA, std::string("iteration capture: ") + cudaGetErrorString(ce));
  }
  return RT_OK;
}

// (a sharded solve exchanges blocks between iterations from the host: one at a time)
static inline bool can_speculate(const rtcur_engine* e) { return e->spec_ok && !e->shard; }

extern "C" int rtcur_engine_can_speculate(rtcur_engine* e) { return e && can_speculate(e) ? 1 : 0; }

extern "C" int rtcur_engine_set_eps(rtcur_engine* e, double eps) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  e->eps = eps;
  return RT_OK;
}

// a state slot nothing still reads: not the latest iterate, its threshold state, the
// shadow, nor (while a speculative iteration may be cancelled) what the iteration before
// it would fall back to
static int alloc_slot(rtcur_engine* e) {
  for (int t = 0; t < RT_STATE_SLOTS; ++t) {
    const int s = (e->alloc_rr + t) % RT_STATE_SLOTS;
    if (s == e->cur || s == e->prev || s == e->shadow) continue;
    if (e->snap_valid && (s == e->snap.cur || s == e->snap.prev || s == e->snap.shadow)) continue;
    e->alloc_rr = (s + 1) % RT_STATE_SLOTS;
    return s;
  }
  return -1;
}

static void take_snapshot(rtcur_engine* e) {
  auto& sn = e->snap;
  sn.cur = e->cur; sn.prev = e->prev; sn.act = e->act; sn.stg = e->stg; sn.sample_epoch = e->sample_epoch;
  for (int i = 0; i < RT_STATE_SLOTS; ++i) sn.w_epoch[i] = e->w_epoch[i];
  sn.shadow = e->shadow; sn.shadow_of = e->shadow_of; sn.shadow_epoch = e->shadow_epoch; sn.alloc_rr = e->alloc_rr;
  sn.zeta_last = e->zeta_last;
  for (int s = 0; s < RT_SAMPLE_SLOTS; ++s) sn.xi_valid[s] = e->xi_valid[s];
  e->snap_valid = true;
  e->snap_seq = e->launch_seq + 1;
}

extern "C" int rtcur_engine_iterate_async(rtcur_engine* e, double zeta, int first) {
  if (!e || !e->sampled) return fail(RT_ERR_VALUE, "engine has no sample");
  if (e->npending >= 2) return fail(RT_ERR_VALUE, "two iterations already in flight");
  const bool spec = e->npending == 1;
  if (spec && (first || !can_speculate(e))) return fail(RT_ERR_VALUE, "previous iteration not waited for");
  if (!(zeta >= 0.0)) return fail(RT_ERR_VALUE, "threshold must be nonnegative");
  if (spec) take_snapshot(e);   // what rtcur_engine_iterate_cancel restores
  else e->snap_valid = false;
  e->cur_seq = ++e->launch_seq;
  if (e->staging_on_side) {   // the prefetched sample's staging must be complete
    CK(cudaStreamWaitEvent(e->st, e->side_ev, 0));
    e->staging_on_side = false;
  }
  if (e->stg >= 0) {   // the staged sample (set_sample + gather) becomes the active one
    e->act = e->stg;
    e->stg = -1;
    e->sample_epoch++;
  }
  // everything before this iteration (the previous iteration, exports) is what a
  // prefetch into the other sample slot must wait for
  CK(cudaEventRecord(e->pre_ev, e->st));
  if (first) {
    if (int st = flush_tail(e)) return st;   // (a previous solve's)
    e->cur = e->prev = e->shadow = -1;
    e->r_mode = false;
    e->join_needed = false;
    if (e->prof_on && getenv("RTCUR_PROF_TIMELINE")) {
      if (!e->tl_base) cudaEventCreate(&e->tl_base);
      CK(cudaEventRecord(e->tl_base, e->st));
    }
    CK(cudaMemsetAsync(stop_flag(e), 0, 4, e->st));   // a new solve: the previous one's stop flag
  }
  // the threshold state: the shadow (a copy of the latest iterate evaluated on the sample
  // that just became active) when the side stream prepared one, else the latest iterate
  // itself, re-evaluated in place when the sample moved
  const bool use_shadow = e->cur >= 0 && e->shadow >= 0 && e->shadow_of == e->cur && e->shadow_epoch == e->sample_epoch;
  const int st_slot = e->cur < 0 ? -1 : (use_shadow ? e->shadow : e->cur);
  const double* st_s = st_slot >= 0 ? e->state(st_slot) : nullptr;
  const bool reeval = st_slot >= 0 && !use_shadow && e->w_epoch[e->cur] != e->sample_epoch;
  // an in-place re-evaluation overwrites the W the previous iteration's error pass reads;
  // in RTCUR-R mode that tail also produces the W this iteration would read when it does
  // not have a shadow; and without graphs nothing is deferred: the tail goes first, in
  // stream order
  if (reeval || !e->use_graphs || (e->r_mode && !use_shadow))
    if (int st = flush_tail(e)) return st;
  if (use_shadow) e->shadow = -1;   // consumed: it is this iteration's threshold state from here on
  const int keep_prev = e->prev;
  e->prev = st_slot;                // (so the allocator keeps it)
  const int newslot = alloc_slot(e);
  e->prev = keep_prev;
  if (newslot < 0) return fail(RT_ERR_VALUE, "no free iterate slot");
  const int par = e->par;
  e->cur_par = par;
  e->zeta_last = zeta;
  e->h_pinned[200 + 4 * par] = zeta;   // read by the iteration's first (memcpy) node
  e->h_pinned[200 + 4 * par + 1] = e->eps;
  e->zetap_cur = e->at<double>(e->P.o_zeta + 32 * par);
  // the iteration's kernels test the stop flag (Geom::stop is copied into every launch)
  e->P.g.stop = stop_flag(e);
  int st = RT_OK;
  auto leave = [&](int code) {
    e->zetap_cur = nullptr;
    e->P.g.stop = nullptr;
    e->cur_seq = 0;
    return code;
  };
  if (e->use_graphs) {
    const unsigned long long key = (unsigned long long)(e->cur + 1) | ((unsigned long long)(st_slot + 1) << 3) |
                                   ((unsigned long long)newslot << 6) | ((unsigned long long)e->act_slot() << 14) |
                                   ((unsigned long long)reeval << 10) |
                                   ((unsigned long long)fiber_refresh_pending(e) << 11) |
                                   ((unsigned long long)par << 12) | ((unsigned long long)e->r_mode << 13) |
                                   ((unsigned long long)(e->prof_on ? (e->prof_mask & kIterPhases) : 0u) << 16);
    auto it = e->graphs->find(key);
    if (it == e->graphs->end()) {
      GraphEntry ge;
      st = capture_iteration(e, ge, st_s, newslot, reeval, par);
      if (st != RT_OK) return leave(st);
      it = e->graphs->emplace(key, std::move(ge)).first;
    }
    st = launch_entry(e, it->second);
    if (st) return leave(st);
    rtcur_launch_counter_add(it->second.nkernels);   // the graph's kernels run now
    // the tail is held back: the next iteration enqueues it under its eigensolver, or
    // iterate_wait sends it out in stream order
    if (int fst = flush_tail(e)) return leave(fst);   // (one not taken at CUT_EIG: cannot happen, kept for safety)
    e->tail_pending.ge = &it->second;
    e->tail_pending.par = par;
    e->tail_pending.seq = e->cur_seq;
    e->tail_pending.valid = true;
    const bool defer = tail_deferred(e);
    if (!defer)
      if (int fst = flush_tail(e)) return leave(fst);
  } else {
    st = iterate_main(e, st_s, newslot, reeval, par);
    if (st == RT_OK) st = iterate_tail(e, st_s, newslot, par);
    if (st) return leave(st);
    CK(cudaEventRecord(e->done[par], e->st));
  }
  leave(RT_OK);
  CK(cudaEventRecord(e->main_ev, e->st));
  if (reeval) e->w_epoch[e->cur] = e->sample_epoch;
  e->w_epoch[newslot] = e->sample_epoch;
  e->prev = st_slot;
  e->cur = newslot;
  e->cur_of_seq = e->launch_seq;
  e->pend_par[e->npending++] = par;
  e->par ^= 1;
  return RT_OK;
}

extern "C" int rtcur_engine_iterate_wait(rtcur_engine* e, double* sums, int* flags) {
  if (!e || e->npending < 1) return fail(RT_ERR_VALUE, "no iteration in flight");
  const int par = e->pend_par[0];
  // its tail is still held back when no iteration was enqueued behind it
  if (e->npending == 1 && e->tail_pending.valid && e->tail_pending.par == par)
    if (int st = flush_tail(e)) return st;
  e->pend_par[0] = e->pend_par[1];
  e->npending--;
  CK(cudaEventSynchronize(e->done[par]));
  prof_flush(e);
  const Plan& P = e->P;
  const char* hr = reinterpret_cast<const char*>(e->h_pinned + par * RES_SLOT);
  int nonfinite;
  memcpy(&nonfinite, hr + (P.o_nonfinite - P.o_sums), 4);
  memcpy(&e->last_stop, hr + (P.o_nonfinite + 4 - P.o_sums), 4);
  if (nonfinite) return fail(RT_ERR_VALUE, "truncated_svd input contains non-finite entries");
  if (sums) memcpy(sums, hr, 2 * P.g.nblk * 8);
  if (flags) memcpy(flags, hr + (P.o_flags - P.o_sums), P.g.n * 4);
  return RT_OK;
}

// 1 when the device-side stop rule fired for the iteration waited for last (its
// sampled relative error <= eps): a speculative iteration enqueued behind it ran nothing.
extern "C" int rtcur_engine_last_stop(rtcur_engine* e) { return e ? e->last_stop : 0; }

// Forget the speculative iteration (enqueued while its predecessor was in flight, after
// that predecessor met the stop rule: its kernels returned at once): the engine's
// bookkeeping returns to the predecessor, which stays the exportable iterate.
extern "C" int rtcur_engine_iterate_cancel(rtcur_engine* e) {
  if (!e || e->npending != 1 || !e->snap_valid) return fail(RT_ERR_VALUE, "no speculative iteration to cancel");
  const auto& sn = e->snap;
  e->cur = sn.cur; e->prev = sn.prev; e->act = sn.act; e->stg = sn.stg; e->sample_epoch = sn.sample_epoch;
  for (int i = 0; i < RT_STATE_SLOTS; ++i) e->w_epoch[i] = sn.w_epoch[i];
  e->shadow = sn.shadow; e->shadow_of = sn.shadow_of; e->shadow_epoch = sn.shadow_epoch; e->alloc_rr = sn.alloc_rr;
  e->zeta_last = sn.zeta_last;
  for (int s = 0; s < RT_SAMPLE_SLOTS; ++s) e->xi_valid[s] = sn.xi_valid[s];
  e->snap_valid = false;
  e->npending = 0;
  e->tail_pending.valid = false;   // its tail is never enqueued
  // its profiled phases measured empty segments: drop them
  {
    std::vector<ProfPair> keep;
    for (auto& p : *e->prof_pending) {
      if (p.seq != e->snap_seq) {
        keep.push_back(p);
        continue;
      }
      if (!p.owned) continue;
      e->prof_pool->push_back(p.b);
      e->prof_pool->push_back(p.e);
    }
    e->prof_pending->swap(keep);
  }
  for (int ph = 0; ph < RT_NPHASE; ++ph)
    if (e->prof_open[ph]) {
      e->prof_pool->push_back(e->prof_open[ph]);
      e->prof_open[ph] = nullptr;
    }
  return RT_OK;
}

extern "C" int rtcur_engine_iterate(rtcur_engine* e, double zeta, int first, double* sums, int* flags) {
  int st = rtcur_engine_iterate_async(e, zeta, first);
  if (st) return st;
  return rtcur_engine_iterate_wait(e, sums, flags);
}

extern "C" int rtcur_engine_export_blocks(rtcur_engine* e, double* s_blocks, double* clean_blocks, double* l_blocks) {
  if (!e || e->cur < 0) return fail(RT_ERR_VALUE, "no iterate to export");
  const double* st_s = e->prev >= 0 ? e->state(e->prev) : nullptr;
  int st = run_block_pass(e, st_s, l_blocks ? e->state(e->cur) : nullptr, e->zeta_last, false, s_blocks,
                          clean_blocks, l_blocks, false, PH_EXPORT);
  if (st) return st;
  CK(cudaStreamSynchronize(e->st));
  prof_flush(e);
  return RT_OK;
}

extern "C" int rtcur_engine_export_cur(rtcur_engine* e, double* const* U, double* const* sigma, double* const* V,
                                       double* const* A, double* G) {
  if (!e || e->cur < 0) return fail(RT_ERR_VALUE, "no iterate to export");
  const Plan& P = e->P;
  const Geom& g = P.g;
  const double* sto = e->state(e->cur);
  // every piece through one page-locked staging buffer (kept by the engine): the copies
  // are truly asynchronous, one synchronisation, then plain host copies out (a D2H into
  // pageable memory is staged and synchronous: 13 of them cost ~0.35 ms at config 1)
  struct Piece { double* dst; const void* src; size_t bytes; };
  std::vector<Piece> pieces;
  for (int m = 0; m < g.n; ++m) {
    if (U && U[m]) pieces.push_back({U[m], e->ws + P.o_U[m], (size_t)(g.nrows[m] * g.rank[m] * 8)});
    if (sigma && sigma[m]) pieces.push_back({sigma[m], e->ws + P.o_sig[m], (size_t)(g.rank[m] * 8)});
    if (V && V[m]) pieces.push_back({V[m], e->ws + P.o_V[m], (size_t)(g.ncols[m] * g.rank[m] * 8)});
    if (A && A[m]) pieces.push_back({A[m], sto + g.a_off[m], (size_t)(g.dim[m] * g.rank[m] * 8)});
  }
  if (G) pieces.push_back({G, sto, (size_t)(g.gsize * 8)});
  size_t total = 0;
  for (auto& pc : pieces) total += (pc.bytes + 63) & ~(size_t)63;
  if (total > e->h_export_bytes) {
    if (e->h_export) cudaFreeHost(e->h_export);
    e->h_export = nullptr;
    e->h_export_bytes = 0;
    CK(cudaMallocHost(&e->h_export, total));
    e->h_export_bytes = total;
  }
  size_t off = 0;
  for (auto& pc : pieces) {
    CK(cudaMemcpyAsync(e->h_export + off, pc.src, pc.bytes, cudaMemcpyDeviceToHost, e->st));
    off += (pc.bytes + 63) & ~(size_t)63;
  }
  CK(cudaStreamSynchronize(e->st));
  off = 0;
  for (auto& pc : pieces) {
    memcpy(pc.dst, e->h_export + off, pc.bytes);
    off += (pc.bytes + 63) & ~(size_t)63;
  }
  return RT_OK;
}

extern "C" int64_t rtcur_engine_full_scratch_bytes(rtcur_engine* e) {
  if (!e) return 0;
  i64 q = 1;
  for (int m = 1; m < e->P.g.n; ++m) q *= e->P.g.dim[m];
  return q * e->P.g.rank[0] * 8 + 16;   // +16: k_full_tma reads Tf rows in 16-byte units
}

extern "C" int rtcur_engine_full_output(rtcur_engine* e, double zeta, void* L_dev, void* S_dev, double* tf_dev,
                                        double* sums) {
  if (!e || e->cur < 0) return fail(RT_ERR_VALUE, "no iterate");
  if (!(zeta >= 0.0)) return fail(RT_ERR_VALUE, "threshold must be nonnegative");
  const Plan& P = e->P;
  const Geom& g = P.g;
  IndexPtrs ip = make_ip(e);
  double* sto = e->state(e->cur);
  i64 ncols = 1;
  for (int m = 1; m < g.n; ++m) ncols *= g.dim[m];
  prof_begin(e, PH_WCOLS);
  {
    i64 Pm[RT_MAX_MODES];
    for (int m = 0; m < g.n; ++m) Pm[m] = g.dim[m];
    int st = run_wchain(e, sto, nullptr, Pm, tf_dev);   // Tf = G x_{m>=2} A_m over the full tensor
    if (st) return st;
  }
  (void)ip;
  prof_end(e, PH_WCOLS);
  FullArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.X = e->X;   // may be null: reconstruction only (x = 0)
  fa.dtype = P.dtype;
  fa.lo = e->lo;
  fa.hi = e->hi;
  fa.ncols = ncols;
  fa.A1 = sto + g.a_off[0];
  fa.d1 = g.dim[0];
  fa.r1 = g.rank[0];
  fa.Tf = tf_dev;
  fa.zeta = zeta;
  fa.L = L_dev;
  fa.S = S_dev;
  fa.partial = e->at<double>(P.o_fpart);
  fa.sums = e->at<double>(P.o_sums);
  fa.counter = e->at<unsigned int>(P.o_counters) + 32;
  const int grid = 148 * 8;
  prof_begin(e, PH_FULL);
  const int tma = full_tma_launch(fa, grid, e->st);
  if (tma < 0) return fail(RT_ERR_CUDA, std::string("k_full_tma: ") + cudaGetErrorString((cudaError_t)(-tma)));
  if (tma == 0) {
    if (P.dtype == 0) k_full<double><<<grid, 256, 0, e->st>>>(fa);
    else k_full<float><<<grid, 256, 0, e->st>>>(fa);
  }
  LAUNCH_CHECK();
  prof_end(e, PH_FULL);
  CK(cudaMemcpyAsync(e->h_pinned, fa.sums, 16, cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  prof_flush(e);
  if (sums) memcpy(sums, e->h_pinned, 16);
  return RT_OK;
}

// internal diagnostics: clock64 phase marks of the last eigensolver launch (8 per mode)
extern "C" int rtcur_engine_debug_marks(rtcur_engine* e, int64_t* out, int n) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  CK(cudaStreamSynchronize(e->st));
  CK(cudaMemcpy(out, e->ws + e->P.o_dbg, sizeof(int64_t) * std::min(n, 8 * RT_MAX_MODES), cudaMemcpyDeviceToHost));
  if (n >= 8 * RT_MAX_MODES + RT_MAX_MODES) {
    int f[RT_MAX_MODES];
    CK(cudaMemcpy(f, e->ws + e->P.o_fast, sizeof(int) * RT_MAX_MODES, cudaMemcpyDeviceToHost));
    for (int m = 0; m < RT_MAX_MODES; ++m) out[8 * RT_MAX_MODES + m] = f[m];
  }
  return RT_OK;
}

extern "C" int rtcur_engine_set_graphs(rtcur_engine* e, int on) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  if (e->npending) return fail(RT_ERR_VALUE, "iteration in flight");
  e->use_graphs = on != 0;
  return RT_OK;
}

extern "C" int rtcur_engine_profile_phases(rtcur_engine* e, uint32_t mask) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  CK(cudaStreamSynchronize(e->st));
  prof_flush(e);
  e->prof_mask = mask ? mask : ~0u;
  return RT_OK;
}

extern "C" int rtcur_engine_profile(rtcur_engine* e, int on) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  CK(cudaStreamSynchronize(e->st));
  prof_flush(e);
  e->prof_on = on != 0;
  if (on) e->prof_mask = e->prof_mask ? e->prof_mask : ~0u;
  return RT_OK;
}

extern "C" int rtcur_engine_profile_read(rtcur_engine* e, double* ms, int64_t* counts, int nphase, int reset) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  CK(cudaStreamSynchronize(e->st));
  prof_flush(e);
  for (int i = 0; i < nphase && i < RT_NPHASE; ++i) {
    if (ms) ms[i] = e->prof_ms[i];
    if (counts) counts[i] = e->prof_cnt[i];
  }
  if (reset)
    for (int i = 0; i < RT_NPHASE; ++i) { e->prof_ms[i] = 0.0; e->prof_cnt[i] = 0; }
  return RT_OK;
}

// ------------------------------------------------------------------ host helpers

// Append to out[0..nout) the values of batch[0..nb) not seen before, in order of
// first occurrence (seen: population-byte bitmap kept by the caller).  This is
// the deduplication of the reference's iid draw (fiber_cur.py:202-208:
// np.unique(..., return_index=True) then merged[np.sort(first)]) in O(n); the
// random stream itself stays numpy's Generator.integers.
// numpy Generator.integers(0, population, size=m, dtype=int64) for population <=
// 2^32 - 1: random_bounded_uint64_fill -> buffered_bounded_lemire_uint32 on the
// bit generator's own next_uint32 (numpy/random/src/distributions), reproduced
// here call for call so the stream (and the generator state afterwards) is the
// one numpy produces.
typedef uint32_t (*rt_next_u32)(void*);
static inline uint32_t rt_lemire32(void* st, rt_next_u32 next, uint32_t rng) {
  const uint32_t rng_excl = rng + 1;
  uint64_t m = (uint64_t)next(st) * rng_excl;
  uint32_t leftover = (uint32_t)m;
  if (leftover < rng_excl) {
    const uint32_t threshold = (UINT32_MAX - rng) % rng_excl;
    while (leftover < threshold) {
      m = (uint64_t)next(st) * rng_excl;
      leftover = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

// The reference's without-replacement draw (fiber_cur.py:197-208, iid branch):
//   out = []; while len(out) < k: batch = integers(0, pop, need + need // 2 + 16);
//   keep the first occurrence of each value in order; return sort(out[:k]) + 1
// natively, drawing from numpy's bit generator (state + next_uint32 of
// Generator.bit_generator.ctypes) so the consumed stream is bit-identical.
// seen: (population + 63) / 64 zeroed words, a membership bitmap (left zeroed);
// out: >= 3k + 32 entries.  Returns k with out[0..k) the sorted 1-based sample,
// or < 0 on a bad argument.
extern "C" int64_t rtcur_draw_distinct(void* bitgen_state, void* next_uint32, int64_t population, int64_t k,
                                       uint64_t* seen, int64_t* out, int64_t out_cap) {
  if (!bitgen_state || !next_uint32 || !seen || !out) return -1;
  if (population < 2 || population > (int64_t)0xFFFFFFFFLL || k < 1 || k >= population || out_cap < 3 * k + 32)
    return -1;
  rt_next_u32 next = reinterpret_cast<rt_next_u32>(next_uint32);
  const uint32_t rng = (uint32_t)(population - 1);
  int64_t nout = 0;
  while (nout < k) {
    const int64_t need = k - nout;
    const int64_t m = need + need / 2 + 16;   // <= 1.5 k + 16: nout stays below 3k + 32
    for (int64_t t = 0; t < m; ++t) {
      const uint32_t v = rt_lemire32(bitgen_state, next, rng);
      uint64_t& w = seen[v >> 6];
      const uint64_t bit = 1ull << (v & 63);
      if (!(w & bit)) {
        w |= bit;
        out[nout++] = v;
      }
    }
  }
  // keep the first k (draw order), then sort them
  for (int64_t i = k; i < nout; ++i) seen[out[i] >> 6] &= ~(1ull << (out[i] & 63));
  const int64_t words = (population + 63) >> 6;
  if (words <= 16 * k) {
    // dense: the bitmap scan yields them sorted (and clears the bitmap)
    int64_t o = 0;
    for (int64_t wi = 0; wi < words && o < k; ++wi) {
      uint64_t w = seen[wi];
      if (!w) continue;
      seen[wi] = 0;
      while (w) {
        const int b = __builtin_ctzll(w);
        out[o++] = (wi << 6) + b + 1;
        w &= w - 1;
      }
    }
    return k;
  }
  for (int64_t i = 0; i < k; ++i) seen[out[i] >> 6] = 0;   // (only the first k bits remained set)
  // sparse: LSD radix sort of the k values (< 2^32), 4 passes of 8 bits through out[k..2k)
  int64_t* a = out;
  int64_t* b = out + k;
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 8 * pass;
    int64_t cnt[257];
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < k; ++i) cnt[((a[i] >> sh) & 255) + 1]++;
    for (int d = 0; d < 256; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < k; ++i) b[cnt[(a[i] >> sh) & 255]++] = a[i];
    std::swap(a, b);
  }
  // 4 passes: the sorted run is back in out[0..k)
  for (int64_t i = 0; i < k; ++i) out[i] += 1;
  return k;
}

extern "C" int64_t rtcur_append_distinct(int64_t* out, int64_t nout, const int64_t* batch, int64_t nb,
                                         unsigned char* seen, int64_t population) {
  for (int64_t i = 0; i < nb; ++i) {
    const int64_t v = batch[i];
    if (v < 0 || v >= population) return -1;
    if (!seen[v]) {
      seen[v] = 1;
      out[nout++] = v;
    }
  }
  return nout;
}

// Synthetic instance on a mode-1 slab (see rtcur_b200.h).  mode 0: *sum_abs = sum |L|
// over the slab; mode 1: X = L + S.  scratch: >= 2 * 148 * 8 doubles + 64 bytes.
extern "C" int rtcur_generate_tucker(const double* Y1, const double* Tf, int64_t d1, int r1, int64_t lo, int64_t hi,
                                     int64_t ncols, int mode, uint64_t seed, double alpha, double cmu, int dtype,
                                     void* X, double* scratch, double* sum_abs, void* stream) {
  if (lo < 0 || hi <= lo || hi > d1 || r1 < 1 || ncols < 1) return fail(RT_ERR_VALUE, "bad generator arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = 148 * 8;
  double* partial = scratch;
  double* outs = scratch + grid;
  unsigned int* counter = reinterpret_cast<unsigned int*>(scratch + grid + 1);
  if (mode == 0) CK(cudaMemsetAsync(counter, 0, 4, st));
  if (dtype == 0)
    k_gen_tucker<double><<<grid, 256, 0, st>>>(Y1, Tf, d1, r1, lo, hi, ncols, mode, seed, alpha, cmu, (double*)X,
                                              partial, outs, counter);
  else
    k_gen_tucker<float><<<grid, 256, 0, st>>>(Y1, Tf, d1, r1, lo, hi, ncols, mode, seed, alpha, cmu, (float*)X,
                                             partial, outs, counter);
  LAUNCH_CHECK();
  if (mode == 0) {
    CK(cudaMemcpyAsync(sum_abs, outs, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return RT_OK;
}

// sum |x| in a fixed order: per-CTA grid-stride partial sums, then one CTA adds the
// partials in CTA order (deterministic run to run).
__global__ void k_abs_sum_part(const double* __restrict__ x, i64 n, double* __restrict__ part) {
  __shared__ double red[8];
  double s = 0.0;
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < n; k += (i64)gridDim.x * blockDim.x) s += fabs(x[k]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_abs_sum_final(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int k = threadIdx.x; k < np; k += blockDim.x) s += part[k];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

extern "C" int rtcur_abs_sum(const double* x, int64_t n, double* scratch, double* out, void* stream) {
  if (!x || !scratch || !out || n < 0) return fail(RT_ERR_VALUE, "bad abs-sum arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int np = 148 * 4;
  k_abs_sum_part<<<np, 256, 0, st>>>(x, n, scratch);
  LAUNCH_CHECK();
  k_abs_sum_final<<<1, 256, 0, st>>>(scratch, np, scratch + np);
  LAUNCH_CHECK();
  CK(cudaMemcpyAsync(out, scratch + np, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return RT_OK;
}

// Outliers of the reference generator (synth.py:101-121): value_k = low + (high - low) * u_k
// with low = -mu, high = mu, rounded step by step like numpy's Generator.uniform (no FMA);
// S[pos_k] = value_k and X[pos_k] += value_k (fp64, X holding L: x = low + sparse).
__global__ void k_scatter_outliers(double* __restrict__ X, const int64_t* __restrict__ pos,
                                   const double* __restrict__ u, i64 count, double mu, double* __restrict__ S) {
  const double lo = -mu, span = __dadd_rn(mu, mu);
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < count; k += (i64)gridDim.x * blockDim.x) {
    const double v = __dadd_rn(lo, __dmul_rn(span, u[k]));
    const i64 p = pos[k];
    X[p] = __dadd_rn(X[p], v);
    if (S) S[p] = v;
  }
}

extern "C" int rtcur_scatter_outliers(double* X, const int64_t* pos, const double* u, int64_t count, double mu,
                                      double* S, void* stream) {
  if (!X || count < 0 || (count > 0 && (!pos || !u))) return fail(RT_ERR_VALUE, "bad outlier arguments");
  if (count == 0) return RT_OK;
  k_scatter_outliers<<<(unsigned)std::min<i64>(cdiv(count, 256), 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      X, pos, u, count, mu, S);
  LAUNCH_CHECK();
  return RT_OK;
}

// ---- dense HOSVD alternating projections (reference.py:132-193), full-tensor passes
// S = HT(X - L, zeta) (strict |.| > zeta keep, solver.py:195-199) and C = X - S, one pass.
__global__ void k_ap_threshold(const double* __restrict__ X, const double* __restrict__ L, i64 n, double zeta,
                               double* __restrict__ S, double* __restrict__ C) {
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < n; k += (i64)gridDim.x * blockDim.x) {
    const double x = X[k];
    const double s = hard_thr(x - (L ? L[k] : 0.0), zeta);
    S[k] = s;
    C[k] = x - s;
  }
}
// fixed-order sum of (X - L - S)^2 (and X^2): per-CTA partials, one CTA adds them in order
__global__ void k_ap_resid_part(const double* __restrict__ X, const double* __restrict__ L,
                                const double* __restrict__ S, i64 n, double* __restrict__ part) {
  __shared__ double red[8];
  double e2 = 0.0, x2 = 0.0;
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < n; k += (i64)gridDim.x * blockDim.x) {
    const double x = X[k];
    const double rr = x - L[k] - S[k];
    e2 = fma(rr, rr, e2);
    x2 = fma(x, x, x2);
  }
  e2 = block_sum(e2, red);
  x2 = block_sum(x2, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = e2;
    part[2 * blockIdx.x + 1] = x2;
  }
}
__global__ void k_ap_resid_final(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double red[8];
  double e2 = 0.0, x2 = 0.0;
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    e2 += part[2 * k];
    x2 += part[2 * k + 1];
  }
  e2 = block_sum(e2, red);
  x2 = block_sum(x2, red);
  if (threadIdx.x == 0) {
    out[0] = e2;
    out[1] = x2;
  }
}

extern "C" int rtcur_abs_max(const void* x, int dtype, int64_t n, double* scratch, double* out, void* stream) {
  if (!x || !scratch || !out || n < 0 || (dtype != 0 && dtype != 1)) return fail(RT_ERR_VALUE, "bad abs-max arguments");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* d = reinterpret_cast<unsigned long long*>(scratch);
  CK(cudaMemsetAsync(d, 0, 8, st));
  if (n > 0) {
    if (dtype == 0) k_absmax<double><<<148 * 8, 256, 0, st>>>((const double*)x, n, d);
    else k_absmax<float><<<148 * 8, 256, 0, st>>>((const float*)x, n, d);
    LAUNCH_CHECK();
  }
  unsigned long long bits = 0;
  CK(cudaMemcpyAsync(&bits, d, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  memcpy(out, &bits, 8);
  return RT_OK;
}

extern "C" int rtcur_ap_threshold(const double* X, const double* L, int64_t n, double zeta, double* S, double* C,
                                  void* stream) {
  if (!X || !S || !C || n < 0 || !(zeta >= 0.0)) return fail(RT_ERR_VALUE, "bad threshold arguments");
  if (n == 0) return RT_OK;
  k_ap_threshold<<<(unsigned)std::min<i64>(cdiv(n, 256), 148 * 16), 256, 0, (cudaStream_t)stream>>>(X, L, n, zeta, S,
                                                                                                    C);
  LAUNCH_CHECK();
  return RT_OK;
}

extern "C" int rtcur_ap_residual(const double* X, const double* L, const double* S, int64_t n, double* scratch,
                                 double* sums, void* stream) {
  if (!X || !L || !S || !scratch || !sums || n < 0) return fail(RT_ERR_VALUE, "bad residual arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int np = 148 * 4;
  k_ap_resid_part<<<np, 256, 0, st>>>(X, L, S, n, scratch);
  LAUNCH_CHECK();
  k_ap_resid_final<<<1, 256, 0, st>>>(scratch, np, scratch + 2 * np);
  LAUNCH_CHECK();
  CK(cudaMemcpyAsync(sums, scratch + 2 * np, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return RT_OK;
}

// ------------------------------------------------------------------ kernel-level plug

extern "C" int rtcur_gather_columns(const void* flat, int dtype, int64_t flat_len, const int64_t* bases_dev,
                                    int64_t ncols, int64_t stride, int64_t length, double* out, void* stream) {
  if (stride < 1 || length < 1) return fail(RT_ERR_VALUE, "stride and length must be >= 1");
  if (ncols == 0) return RT_OK;
  // bounds (py_kernels.py:242-251): check on the device copy via a host round trip of min/max
  std::vector<int64_t> b(ncols);
  CK(cudaMemcpyAsync(b.data(), bases_dev, ncols * 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  for (int64_t c = 0; c < ncols; ++c)
    if (b[c] < 0 || b[c] + (length - 1) * stride >= flat_len)
      return fail(RT_ERR_VALUE, "gather out of range: base " + std::to_string(b[c]));
  const i64 n = ncols * length;
  k_gather_columns<<<(unsigned)std::min<i64>(cdiv(n, 256), 4096), 256, 0, (cudaStream_t)stream>>>(
      flat, dtype, bases_dev, ncols, stride, length, out);
  LAUNCH_CHECK();
  return RT_OK;
}

extern "C" int rtcur_hard_threshold(const double* a, int64_t n, double zeta, double* out, void* stream) {
  if (!(zeta >= 0.0)) return fail(RT_ERR_VALUE, "threshold must be nonnegative");
  if (n == 0) return RT_OK;
  k_hard_threshold<<<(unsigned)std::min<i64>(cdiv(n, 256), 4096), 256, 0, (cudaStream_t)stream>>>(a, n, zeta, out);
  LAUNCH_CHECK();
  return RT_OK;
}

extern "C" int rtcur_truncated_svd(const double* m_dev, int64_t m, int64_t p, int r, double* u_dev, double* s_dev,
                                   double* v_dev, void* stream) {
  if (m < 1 || p < 1) return fail(RT_ERR_VALUE, "truncated_svd needs a nonempty matrix");
  if (r < 1 || r > std::min(m, p)) return fail(RT_ERR_VALUE, "rank outside [1, min(m, p)]");
  cudaStream_t st = (cudaStream_t)stream;
  // Reuse the engine machinery on a one-mode "problem": the intersection is the
  // whole matrix, so plan a 1-mode geometry with |I| = m, |J| = p.
  Plan P;
  memset(&P, 0, sizeof(P));
  P.g.n = 1;
  P.s[0] = std::min(m, p);
  P.l[0] = std::max(m, p);
  P.tall[0] = m > p;
  if (P.s[0] > 235) return fail(RT_ERR_UNSUPPORTED, "min(m, p) > 235 not supported");
  if (r > RT_MAX_RANK) return fail(RT_ERR_UNSUPPORTED, "rank > 32 not supported");
  const i64 s = P.s[0], l = P.l[0];
  P.g.rank[0] = r;
  P.g.nrows[0] = m;
  P.g.ncols[0] = p;
  P.rmax = r;
  P.rb = rbucket(r);
  P.smax = s;
  P.lmax = l;
  P.hchunk = HG_CH;
  P.h_maxchunks = (int)cdiv(l, HG_CH);
  const int nt = (int)cdiv(s, GRAM_T);
  P.gram_maxpairs = nt * (nt + 1) / 2;
  P.gram_cl = (int)std::max<i64>(GRAM_KS, cdiv(cdiv(l, std::max<i64>(1, cdiv(4 * 148, P.gram_maxpairs))), GRAM_KS) * GRAM_KS);
  P.gram_maxchunks = (int)cdiv(l, P.gram_cl);
  P.nb[0] = eig_pick_nb((int)s, r);
  if (P.nb[0] < 1) return fail(RT_ERR_UNSUPPORTED, "matrix too large for the shared-memory eigensolver");
  i64 o = 0;
  auto take = [&](i64 bytes) { i64 rr = o; o += align256(std::max<i64>(bytes, 8)); return rr; };
  P.o_M[0] = take(8);
  P.o_gpart = take((i64)P.gram_maxchunks * P.gram_maxpairs * GRAM_T * GRAM_T * 8);
  P.o_K[0] = take(s * (s + 1) / 2 * 8);
  P.o_E[0] = take(s * r * 8);
  P.o_lam[0] = take(r * 8);
  P.o_Z[0] = take(l * r * 8);
  P.o_hpart[0] = take(cdiv(l, HG_CH) * r * (r + 1) / 2 * 8);
  P.o_H[0] = take(r * r * 8);
  P.o_Q[0] = take(r * r * 8);
  P.o_U[0] = take(m * r * 8);
  P.o_V[0] = take(p * r * 8);
  P.o_sig[0] = take(r * 8);
  P.o_siginv[0] = take(r * 8);
  P.o_perm[0] = take(r * 4);
  P.o_degen[0] = take((r + 1) * 4);
  P.o_flags = take(4);
  P.o_counters = take(64 * 4);
  char* ws = nullptr;
  CK(cudaMallocAsync((void**)&ws, o, st));
  rtcur_engine tmp;
  memset((void*)&tmp, 0, sizeof(tmp));
  tmp.P = P;
  tmp.ws = ws;
  tmp.st = st;
  CK(cudaMemsetAsync(ws + P.o_counters, 0, 64 * 4, st));
  // the SVD kernels take raw pointers: M points straight at the caller's matrix
  int esm = eig_smem_bytes(P, 0);
  {
    int st2 = set_smem_limits_once();
    if (st2) return st2;
  }
  const int zs = (int)(s * (r + ZP_LD) * 8);
  GramArgs ga;
  memset(&ga, 0, sizeof(ga));
  ga.n = 1;
  ga.s[0] = (int)s;
  ga.l[0] = l;
  ga.tall[0] = P.tall[0];
  ga.mrows[0] = m;
  ga.M[0] = m_dev;
  ga.K[0] = tmp.at<double>(P.o_K[0]);
  ga.part = tmp.at<double>(P.o_gpart);
  ga.maxchunks = P.gram_maxchunks;
  ga.maxpairs = P.gram_maxpairs;
  ga.cl = P.gram_cl;
  k_gram_tiles<<<dim3(P.gram_maxpairs, P.gram_maxchunks, 1), 256, 0, st>>>(ga);
  LAUNCH_CHECK();
  k_gram_reduce<<<dim3((unsigned)std::min<i64>(cdiv(s * (s + 1) / 2 * 32, 256), 2048), 1), 256, 0, st>>>(ga);
  LAUNCH_CHECK();
  EigArgs ea;
  memset(&ea, 0, sizeof(ea));
  ea.n = 1;
  ea.s[0] = (int)s;
  ea.r[0] = r;
  ea.K[0] = ga.K[0];
  ea.E[0] = tmp.at<double>(P.o_E[0]);
  ea.lam[0] = tmp.at<double>(P.o_lam[0]);
  ea.nb[0] = P.nb[0];
  ea.full[0] = eig_pick_full((int)s, r);
  ea.lz_stride = 8;   // (no Lanczos capacity is planned here: lz_mcap = 0)
  ea.reg_tridiag = getenv("RTCUR_EIG_REG") ? atoi(getenv("RTCUR_EIG_REG")) : 1;
  {
    const i64 s1[1] = {s};
    if (int st2 = launch_eig(ea, s1, 1, esm, st)) return st2;
  }
  SvdArgs sa = make_svd_args(&tmp);
  sa.M[0] = m_dev;
  unsigned int* hcnt = tmp.at<unsigned int>(P.o_counters) + 16;
  const unsigned gz = (unsigned)cdiv(l, 256);
  DISPATCH_R(P.rb, k_zproj, dim3((unsigned)cdiv(l, ZP_T), 1), 32 * P.rb, zs, st, sa);
  LAUNCH_CHECK();
  const int hsm = (int)((std::max<i64>(HG_CH * r + 512, 7 * (i64)r * r + 3 * r + 8)) * 8);
  k_hgram<3><<<dim3(P.h_maxchunks, 1), 512, hsm, st>>>(sa, hcnt);
  LAUNCH_CHECK();
  DISPATCH_R(P.rb, k_long, dim3(gz, 1), 256, 0, st, sa, hcnt + 8);
  LAUNCH_CHECK();
  // row-major (m x r), (p x r) -> column-major outputs
  std::vector<double> U(m * r), V(p * r), S(r);
  CK(cudaMemcpyAsync(U.data(), sa.U[0], m * r * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(V.data(), sa.V[0], p * r * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(S.data(), sa.sig[0], r * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<double> Uc(m * r), Vc(p * r);
  for (i64 i = 0; i < m; ++i)
    for (int a = 0; a < r; ++a) Uc[i + a * m] = U[i * r + a];
  for (i64 i = 0; i < p; ++i)
    for (int a = 0; a < r; ++a) Vc[i + a * p] = V[i * r + a];
  CK(cudaMemcpyAsync(u_dev, Uc.data(), m * r * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(v_dev, Vc.data(), p * r * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(s_dev, S.data(), r * 8, cudaMemcpyHostToDevice, st));
  CK(cudaFreeAsync(ws, st));
  CK(cudaStreamSynchronize(st));
  return RT_OK;
}
