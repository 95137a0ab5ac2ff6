// shard_xchg.cu -- mode-1 slab sharding: pack this rank's owned sampled entries,
// unpack every rank's packed entries into the replicated compact blocks
// (the reference's per-iteration regather is solver.py:315-322,
// the blocks it builds are solver.py:234-239).  Included by engine.cu.
//
// Ownership (rank p holds X[lo_p:hi_p, ...]): every sampled entry belongs to the
// rank whose slab holds its mode-1 index:
//   core block      (|I_1| x prod|I_m|)  rows I_1 ∩ [lo_p, hi_p): a row band, all columns
//   fiber mode 1    (d_1 x |J_1|)        rows [lo_p, hi_p): a row band, all columns
//   fiber mode k>=2 (d_k x |J_k|)        whole columns whose decoded i_1 lies in the slab
// Packed layout of rank p's segment: blocks in order; inside a block, its owned
// columns in increasing column order, each column's row band contiguous.  One
// all-gather of the packed segments (padded to the largest) moves each sampled
// entry exactly once ((P-1)/P of E*N_blk received per rank), and the unpack
// restores bit-exactly the blocks an unsharded gather would produce.
//
// Per sample slot the host builds (rtcur_engine_shard_plan) a descriptor table
// desc[p][b] = {r0, r1, c0, c1, poff} and, for fiber blocks of modes >= 2, the
// columns ordered by owner (stable), then uploads both; pack and unpack are one
// warp per (rank, owned column) copying its row band with coalesced accesses.

#define SH_DESC 5   // r0, r1, c0, c1, poff

struct ShardOrd {
  i64 off[RT_MAX_BLOCKS];   // offset of block b's column order in ord (-1: identity)
};

struct ShardState {
  int world, rank;
  std::vector<i64> bounds;         // world + 1 mode-1 slab boundaries
  i64 desc_elems, ord_elems;       // per slot: world*nblk*SH_DESC i64, sum_{b>=2} Q_b int32
  i64 ordoff[RT_MAX_BLOCKS];       // offset of block b's column order in ord (-1: identity)
  char* h_plan[2];                 // pinned staging per sample slot
  char* d_plan[2];                 // device copy per sample slot
  cudaEvent_t up_ev[2];            // the slot's plan upload done (staging reusable)
  std::vector<i64> counts[2];      // packed entries per rank, per slot
  i64 bytes() const { return desc_elems * 8 + ord_elems * 4; }
};

template <typename T, bool PACK>
__global__ void __launch_bounds__(256) k_shard_copy(Geom g, const i64* __restrict__ desc, const int* __restrict__ ord,
                                                    ShardOrd so, int p_fixed, T* __restrict__ xb, T* __restrict__ buf,
                                                    i64 maxc) {
  const int p = PACK ? p_fixed : (int)blockIdx.y;
  const i64* dp = desc + (i64)p * g.nblk * SH_DESC;
  i64 ntask = 0;
  for (int b = 0; b < g.nblk; ++b) ntask += dp[b * SH_DESC + 3] - dp[b * SH_DESC + 2];
  const int lane = threadIdx.x & 31;
  const i64 nwarps = (i64)gridDim.x * (blockDim.x >> 5);
  T* seg = PACK ? buf : buf + (i64)p * maxc;
  for (i64 t = (i64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntask; t += nwarps) {
    int b = 0;
    i64 tl = t;
    for (;; ++b) {
      const i64 nc = dp[b * SH_DESC + 3] - dp[b * SH_DESC + 2];
      if (tl < nc) break;
      tl -= nc;
    }
    const i64 r0 = dp[b * SH_DESC + 0], r1 = dp[b * SH_DESC + 1], c0 = dp[b * SH_DESC + 2];
    const i64 poff = dp[b * SH_DESC + 4];
    const i64 rows = r1 - r0;
    const i64 c = so.off[b] >= 0 ? (i64)ord[so.off[b] + c0 + tl] : c0 + tl;
    const BlockDesc& bd = g.blk[b];
    T* cp = xb + bd.off + c * bd.P + r0;
    T* pp = seg + poff + tl * rows;
    for (i64 i = lane; i < rows; i += 32) {
      if (PACK) pp[i] = cp[i];
      else cp[i] = pp[i];
    }
  }
}

static int shard_free(rtcur_engine* e) {
  ShardState* s = e->shard;
  if (!s) return RT_OK;
  for (int k = 0; k < 2; ++k) {
    if (s->up_ev[k]) cudaEventSynchronize(s->up_ev[k]), cudaEventDestroy(s->up_ev[k]);
    if (s->h_plan[k]) cudaFreeHost(s->h_plan[k]);
    if (s->d_plan[k]) cudaFree(s->d_plan[k]);
  }
  delete s;
  e->shard = nullptr;
  return RT_OK;
}

extern "C" int rtcur_engine_set_shards(rtcur_engine* e, int world, int rank, const int64_t* bounds) {
  if (!e) return fail(RT_ERR_VALUE, "null engine");
  const Geom& g = e->P.g;
  if (world < 1 || rank < 0 || rank >= world || !bounds) return fail(RT_ERR_VALUE, "bad shard layout");
  if (bounds[0] != 0 || bounds[world] != g.dim[0]) return fail(RT_ERR_VALUE, "slabs must cover mode 1 exactly");
  for (int p = 0; p < world; ++p)
    if (bounds[p + 1] < bounds[p]) return fail(RT_ERR_VALUE, "slab boundaries must be non-decreasing");
  if (bounds[rank] != e->lo || bounds[rank + 1] != e->hi)
    return fail(RT_ERR_VALUE, "this rank's slab does not match the engine's [lo, hi)");
  CK(cudaStreamSynchronize(e->st));
  shard_free(e);
  ShardState* s = new ShardState();
  s->world = world;
  s->rank = rank;
  s->bounds.assign(bounds, bounds + world + 1);
  s->desc_elems = (i64)world * g.nblk * SH_DESC;
  i64 o = 0;
  for (int b = 0; b < g.nblk; ++b) {
    const BlockDesc& bd = g.blk[b];
    if (!bd.is_core && bd.mode >= 1) {
      s->ordoff[b] = o;
      o += bd.Q;
    } else {
      s->ordoff[b] = -1;
    }
  }
  s->ord_elems = o;
  e->shard = s;
  for (int k = 0; k < 2; ++k) {
    CK(cudaHostAlloc((void**)&s->h_plan[k], (size_t)std::max<i64>(s->bytes(), 8), cudaHostAllocDefault));
    CK(cudaMalloc((void**)&s->d_plan[k], (size_t)std::max<i64>(s->bytes(), 8)));
    CK(cudaEventCreateWithFlags(&s->up_ev[k], cudaEventDisableTiming));
    s->counts[k].assign(world, 0);
  }
  return RT_OK;
}

// plan of the staged sample (the slot the last set_sample wrote); counts[p] =
// entries rank p contributes.  Host work is O(|I_1| + sum_k |J_k| + world * nblk).
extern "C" int rtcur_engine_shard_plan(rtcur_engine* e, int64_t* counts) {
  if (!e || !e->shard) return fail(RT_ERR_VALUE, "no shard layout (rtcur_engine_set_shards)");
  if (!e->sampled) return fail(RT_ERR_VALUE, "no sample set");
  ShardState* s = e->shard;
  const Plan& P = e->P;
  const Geom& g = P.g;
  const int slot = e->stg >= 0 ? e->stg : e->act_slot();
  const int W = s->world;
  CK(cudaEventSynchronize(s->up_ev[slot]));
  const char* hb = reinterpret_cast<const char*>(e->h_idx + (size_t)slot * (e->h_idx_len + 8));
  const int* rows0 = reinterpret_cast<const int*>(hb + (P.o_rows[0] - P.o_rows[0]));
  i64* desc = reinterpret_cast<i64*>(s->h_plan[slot]);
  int* ord = reinterpret_cast<int*>(s->h_plan[slot] + s->desc_elems * 8);
  std::vector<i64> poff(W, 0);
  std::vector<i64> cnt(W + 1);
  const i64 d1 = g.dim[0];
  for (int b = 0; b < g.nblk; ++b) {
    const BlockDesc& bd = g.blk[b];
    if (bd.is_core || bd.mode == 0) {
      for (int p = 0; p < W; ++p) {
        i64 r0, r1;
        if (bd.is_core) {   // rows of I_1 inside the slab: a band of the sorted set
          r0 = std::lower_bound(rows0, rows0 + g.nrows[0], (int)s->bounds[p]) - rows0;
          r1 = std::lower_bound(rows0, rows0 + g.nrows[0], (int)s->bounds[p + 1]) - rows0;
        } else {
          r0 = s->bounds[p];
          r1 = s->bounds[p + 1];
        }
        i64* d = desc + ((i64)p * g.nblk + b) * SH_DESC;
        d[0] = r0;
        d[1] = r1;
        d[2] = 0;
        d[3] = r1 > r0 ? bd.Q : 0;
        d[4] = poff[p];
        poff[p] += (r1 - r0) * d[3];
      }
    } else {   // whole columns, owner from the column's mode-1 index (mode 1 is the fastest other mode)
      const i64* cols = reinterpret_cast<const i64*>(hb + (P.o_cols[bd.mode] - P.o_rows[0]));
      std::fill(cnt.begin(), cnt.end(), 0);
      std::vector<int> own((size_t)bd.Q);
      for (i64 j = 0; j < bd.Q; ++j) {
        const i64 i1 = cols[j] % d1;
        const int p = (int)(std::upper_bound(s->bounds.begin() + 1, s->bounds.end(), i1) - (s->bounds.begin() + 1));
        own[j] = p;
        cnt[p + 1]++;
      }
      for (int p = 0; p < W; ++p) cnt[p + 1] += cnt[p];
      std::vector<i64> fill(cnt.begin(), cnt.end() - 1);
      int* ob = ord + s->ordoff[b];
      for (i64 j = 0; j < bd.Q; ++j) ob[fill[own[j]]++] = (int)j;   // stable: increasing j per owner
      for (int p = 0; p < W; ++p) {
        i64* d = desc + ((i64)p * g.nblk + b) * SH_DESC;
        d[0] = 0;
        d[1] = bd.P;
        d[2] = cnt[p];
        d[3] = cnt[p + 1];
        d[4] = poff[p];
        poff[p] += bd.P * (cnt[p + 1] - cnt[p]);
      }
    }
  }
  for (int p = 0; p < W; ++p) {
    s->counts[slot][p] = poff[p];
    if (counts) counts[p] = poff[p];
  }
  CK(cudaMemcpyAsync(s->d_plan[slot], s->h_plan[slot], (size_t)s->bytes(), cudaMemcpyHostToDevice, e->st));
  CK(cudaEventRecord(s->up_ev[slot], e->st));
  return RT_OK;
}

static int shard_launch(rtcur_engine* e, void* buf, int64_t maxc, bool pack) {
  if (!e || !e->shard) return fail(RT_ERR_VALUE, "no shard layout (rtcur_engine_set_shards)");
  if (!buf) return fail(RT_ERR_VALUE, "null exchange buffer");
  ShardState* s = e->shard;
  const Plan& P = e->P;
  const int slot = e->stg >= 0 ? e->stg : e->act_slot();
  i64 most = 0;
  for (int p = 0; p < s->world; ++p) most = std::max<i64>(most, s->counts[slot][p]);
  if (!pack && maxc < most) return fail(RT_ERR_VALUE, "exchange stride smaller than the largest segment");
  const i64* desc = reinterpret_cast<const i64*>(s->d_plan[slot]);
  const int* ord = reinterpret_cast<const int*>(s->d_plan[slot] + s->desc_elems * 8);
  ShardOrd so;
  for (int b = 0; b < RT_MAX_BLOCKS; ++b) so.off[b] = b < P.g.nblk ? s->ordoff[b] : -1;
  // one warp per owned column: a rank owns at most sum_b Q_b columns
  i64 maxcols = 0;
  for (int b = 0; b < P.g.nblk; ++b) maxcols += P.g.blk[b].Q;
  const unsigned gx = (unsigned)std::max<i64>(1, std::min<i64>(cdiv(maxcols, 8), 148 * 8));
  prof_begin(e, PH_GATHER);
  if (pack) {
    if (P.dtype == 0) k_shard_copy<double, true><<<gx, 256, 0, e->st>>>(P.g, desc, ord, so, s->rank,
                                                                        (double*)e->xb(slot), (double*)buf, maxc);
    else k_shard_copy<float, true><<<gx, 256, 0, e->st>>>(P.g, desc, ord, so, s->rank, (float*)e->xb(slot),
                                                          (float*)buf, maxc);
  } else {
    dim3 grid(gx, (unsigned)s->world);
    if (P.dtype == 0) k_shard_copy<double, false><<<grid, 256, 0, e->st>>>(P.g, desc, ord, so, 0,
                                                                           (double*)e->xb(slot), (double*)buf, maxc);
    else k_shard_copy<float, false><<<grid, 256, 0, e->st>>>(P.g, desc, ord, so, 0, (float*)e->xb(slot),
                                                             (float*)buf, maxc);
    e->xi_valid[slot] = false;   // the blocks changed: intersection copies are refreshed before use
  }
  LAUNCH_CHECK();
  prof_end(e, PH_GATHER);
  return RT_OK;
}

extern "C" int rtcur_engine_shard_pack(rtcur_engine* e, void* send) { return shard_launch(e, send, 0, true); }

extern "C" int rtcur_engine_shard_unpack(rtcur_engine* e, const void* recv, int64_t stride) {
  return shard_launch(e, const_cast<void*>(recv), stride, false);
}
