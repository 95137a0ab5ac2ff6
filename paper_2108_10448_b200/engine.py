"""Python handle on the native RTCUR engine (rtcur_engine_* in include/rtcur_b200.h).

The device workspace is one torch uint8 allocation (torch's caching allocator
owns all HBM); the engine carves it.  Work is issued on the current torch
CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native as nat

__all__ = ["Engine", "acquire_engine"]

# Engines (device workspace + pinned staging + native handle) are pooled per
# problem geometry: creating one costs pinned host allocations and kernel
# attribute setup that would otherwise dominate a short solve.  A pooled engine
# is handed out only when no live SolveResult still references it.
_POOL: dict = {}
_POOL_LOCK = threading.Lock()   # solves may run concurrently on several streams (sweeps)


def acquire_engine(shape, ranks, row_sizes, col_sizes, dtype, slab=None, device=None):
    import torch
    import weakref

    dev = device or torch.device("cuda", torch.cuda.current_device())
    # an engine is bound to the stream it was created on: key the pool by the caller's stream
    key = (tuple(shape), tuple(ranks), tuple(row_sizes), tuple(col_sizes), str(dtype), tuple(slab or (0, shape[0])),
           str(dev), int(torch.cuda.current_stream(dev).cuda_stream))
    eng = None
    with _POOL_LOCK:
        free = _POOL.setdefault(key, [])
        while free:
            ref = free.pop()
            eng = ref() if isinstance(ref, weakref.ref) else ref
            if eng is not None and eng.handle.value:
                break
            eng = None
    if eng is None:
        eng = Engine(shape, ranks, row_sizes, col_sizes, dtype, slab=slab, device=dev)
        # per-iteration CUDA graphs only for solves issued on the device's default stream
        # (concurrent solves on worker streams, sweeps.py, launch directly)
        if torch.cuda.current_stream(dev) != torch.cuda.default_stream(dev):
            nat.check(eng.lib.rtcur_engine_set_graphs(eng.handle, 0))
    eng._pool_key = key
    return eng


def release_engine(eng):
    """Return an engine to the pool (called when the result holding it dies)."""
    key = getattr(eng, "_pool_key", None)
    if key is not None and eng.handle.value:
        eng.unbind_quiet()
        with _POOL_LOCK:
            _POOL.setdefault(key, []).append(eng)


def _parallel_copy(dst, src, parts=8):
    """dst[:] = src with a few threads (numpy releases the GIL for large copies)."""
    n = dst.size
    if n < (1 << 20):
        dst[:] = src
        return
    from concurrent.futures import ThreadPoolExecutor

    bounds = [n * i // parts for i in range(parts + 1)]
    global _COPY_POOL
    if _COPY_POOL is None:
        _COPY_POOL = ThreadPoolExecutor(max_workers=parts)
    list(_COPY_POOL.map(lambda i: np.copyto(dst[bounds[i]:bounds[i + 1]], src[bounds[i]:bounds[i + 1]]),
                        range(parts)))


_COPY_POOL = None

# SolveResult arrays as views of the page-locked D2H target (no second host copy)
PINNED_RESULTS = os.environ.get("RTCUR_PINNED_RESULTS", "1") != "0"


CREATED = [0]   # engines constructed in this process (diagnostics: pooled solves construct none)


def marshal_sample(idx):
    """The C-ABI view of a SampleIndices: per-mode int64 pointer arrays (and the arrays
    they point into).  The RTCUR-R sampler thread builds it right after the draw, so the
    solve loop's set_sample is the native call alone (the marshalling was ~30 us of an
    ~80 us call on the loop's critical host path)."""
    n = len(idx.rows)
    rows = [np.ascontiguousarray(r, dtype=np.int64) for r in idx.rows]
    cols = [np.ascontiguousarray(c, dtype=np.int64) for c in idx.cols]
    rp = (nat.c_i64p * n)(*[r.ctypes.data_as(nat.c_i64p) for r in rows])
    cp = (nat.c_i64p * n)(*[c.ctypes.data_as(nat.c_i64p) for c in cols])
    return rp, cp, (rows, cols)


class Engine:
    def __init__(self, shape, ranks, row_sizes, col_sizes, dtype, slab=None, device=None):
        import torch

        CREATED[0] += 1
        self.lib = nat.load()
        if not torch.cuda.is_available():
            raise RuntimeError("rtcur_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
        self.shape = tuple(int(d) for d in shape)
        self.n = len(self.shape)
        self.ranks = tuple(int(r) for r in ranks)
        self.row_sizes = tuple(int(s) for s in row_sizes)
        self.col_sizes = tuple(int(s) for s in col_sizes)
        self.torch_dtype = dtype
        self.dtype_code = nat.RTCUR_F64 if dtype == torch.float64 else nat.RTCUR_F32
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.slab = slab or (0, self.shape[0])
        dims = nat.i64_array(self.shape)
        rk = nat.i32_array(self.ranks)
        rs = nat.i64_array(self.row_sizes)
        cs = nat.i64_array(self.col_sizes)
        self._args = (dims, rk, rs, cs)
        ws = ctypes.c_int64()
        xo = ctypes.c_int64()
        xn = ctypes.c_int64()
        nat.check(self.lib.rtcur_engine_plan(self.n, dims, rk, rs, cs, self.dtype_code, ctypes.byref(ws),
                                             ctypes.byref(xo), ctypes.byref(xn)))
        self.workspace = torch.empty(int(ws.value) + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        pad = (-base) % 256
        self._ws_ptr = base + pad
        self._ws_off = pad
        self.xblocks_offset = int(xo.value) + pad
        self.nblk_total = int(xn.value)
        self.stream = torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        nat.check(self.lib.rtcur_engine_create(ctypes.byref(h), self.n, dims, rk, rs, cs, self.dtype_code,
                                               ctypes.c_void_p(self._ws_ptr), int(ws.value), int(self.slab[0]),
                                               int(self.slab[1]), ctypes.c_void_p(self.stream.cuda_stream)))
        self.handle = h
        self._x = None
        # compact block geometry (host): core, then fiber blocks
        n = self.n
        self.block_shapes = [(self.row_sizes[0], int(np.prod(self.row_sizes[1:], dtype=np.int64)))]
        self.block_shapes += [(self.shape[k], self.col_sizes[k]) for k in range(n)]
        # element offsets of the blocks in the compact buffer; fiber blocks start
        # 16-byte aligned (TMA bulk copies), as laid out by make_plan in engine.cu
        offs, o = [], 0
        for b, (p, q) in enumerate(self.block_shapes):
            if b >= 1:
                o = (o + 3) & ~3
            offs.append(o)
            o += p * q
        offs.append(o)
        self.block_offsets = offs

    # ------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.rtcur_engine_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ steps
    def xblocks(self):
        """torch view of the compact sampled X blocks (dtype of X) inside the workspace."""
        import torch

        esz = 8 if self.dtype_code == nat.RTCUR_F64 else 4
        off = ctypes.c_int64()
        nat.check(self.lib.rtcur_engine_xblocks_offset(self.handle, ctypes.byref(off)))
        o = int(off.value) + self._ws_off   # offsets are relative to the 256-aligned workspace base
        raw = self.workspace[o:o + self.nblk_total * esz]
        return raw.view(torch.float64 if esz == 8 else torch.float32)

    def bind_mode_copies(self, flat, modes):
        """Build mode-k-fastest copies of the bound tensor for ``modes`` (k >= 1) and
        let the gather read their fibers contiguously; ``modes`` empty: drop them."""
        import torch

        if not modes:
            # (the engine orders anything that reuses the copies' memory after their build)
            nat.check(self.lib.rtcur_engine_bind_mode_copies(self.handle, (ctypes.c_void_p * self.n)()))
            self._mode_copies = {}
            return
        # built on the engine's side stream: the first gather and iteration of the solve do
        # not wait for them (rtcur_engine_build_mode_copy)
        self._mode_copies = {}
        for k in modes:
            out = torch.empty_like(flat)
            nat.check(self.lib.rtcur_engine_build_mode_copy(self.handle, int(k), ctypes.c_void_p(out.data_ptr())))
            self._mode_copies[int(k)] = out

    def bind(self, flat):
        """flat: contiguous CUDA tensor holding this rank's mode-1 slab."""
        self._x = flat
        nat.check(self.lib.rtcur_engine_bind(self.handle, ctypes.c_void_p(flat.data_ptr())))

    def unbind_quiet(self):
        self._x = None
        self.lib.rtcur_engine_bind(self.handle, ctypes.c_void_p(0))

    def unbind(self):
        self._x = None
        nat.check(self.lib.rtcur_engine_bind(self.handle, ctypes.c_void_p(0)))

    def absmax(self) -> float:
        out = ctypes.c_double()
        nat.check(self.lib.rtcur_engine_absmax(self.handle, ctypes.byref(out)))
        return float(out.value)

    def absmax_begin(self):
        """Enqueue the max|X| scan (absmax_end returns it)."""
        nat.check(self.lib.rtcur_engine_absmax_begin(self.handle))

    def absmax_end(self) -> float:
        out = ctypes.c_double()
        nat.check(self.lib.rtcur_engine_absmax_end(self.handle, ctypes.byref(out)))
        return float(out.value)

    def set_sample(self, idx, view=None):
        """Upload a sample's index sets; ``view``: its marshal_sample() result when the
        caller prepared it ahead of time (the RTCUR-R sampler thread does)."""
        rp, cp, keep = view if view is not None else marshal_sample(idx)
        nat.check(self.lib.rtcur_engine_set_sample(self.handle, rp, cp))
        self._keep = keep

    def gather(self):
        nat.check(self.lib.rtcur_engine_gather(self.handle))

    # ------------------------------------------------------------ mode-1 slab exchange (csrc/shard_xchg.cu)
    def set_shards(self, world: int, rank: int, bounds):
        b = nat.i64_array([int(v) for v in bounds])
        nat.check(self.lib.rtcur_engine_set_shards(self.handle, int(world), int(rank), b))
        self.world = int(world)

    def shard_plan(self):
        """Packed entry count of every rank for the staged sample."""
        counts = (ctypes.c_int64 * self.world)()
        nat.check(self.lib.rtcur_engine_shard_plan(self.handle, counts))
        return [int(c) for c in counts]

    def shard_pack(self, send):
        nat.check(self.lib.rtcur_engine_shard_pack(self.handle, ctypes.c_void_p(send.data_ptr())))

    def shard_unpack(self, recv, stride: int):
        nat.check(self.lib.rtcur_engine_shard_unpack(self.handle, ctypes.c_void_p(recv.data_ptr()), int(stride)))

    def iterate(self, zeta: float, first: bool):
        sums = (ctypes.c_double * (2 * (self.n + 1)))()
        flags = (ctypes.c_int32 * self.n)()
        nat.check(self.lib.rtcur_engine_iterate(self.handle, float(zeta), int(bool(first)), sums, flags))
        s = np.frombuffer(sums, dtype=np.float64).copy()
        return s[0::2], s[1::2], tuple(bool(f) for f in flags)

    def iterate_async(self, zeta: float, first: bool):
        nat.check(self.lib.rtcur_engine_iterate_async(self.handle, float(zeta), int(bool(first))))

    def iterate_wait(self):
        sums = (ctypes.c_double * (2 * (self.n + 1)))()
        flags = (ctypes.c_int32 * self.n)()
        nat.check(self.lib.rtcur_engine_iterate_wait(self.handle, sums, flags))
        s = np.frombuffer(sums, dtype=np.float64).copy()
        return s[0::2], s[1::2], tuple(bool(f) for f in flags)

    def reset(self):
        """Start of a solve: restart the engine's slot rings (same graphs every solve)."""
        nat.check(self.lib.rtcur_engine_reset(self.handle))

    def set_eps(self, eps: float):
        """Tolerance of the device-side stop rule (0: it never fires)."""
        nat.check(self.lib.rtcur_engine_set_eps(self.handle, float(eps)))

    def can_speculate(self) -> bool:
        """A second iterate_async may be enqueued behind the one in flight."""
        return bool(self.lib.rtcur_engine_can_speculate(self.handle))

    def last_stop(self) -> bool:
        """The device's stop decision for the iteration waited for last."""
        return bool(self.lib.rtcur_engine_last_stop(self.handle))

    def iterate_cancel(self):
        """Drop the speculative iteration (its predecessor met the stop rule)."""
        nat.check(self.lib.rtcur_engine_iterate_cancel(self.handle))

    def export_blocks(self, want_s=True, want_clean=True, want_l=False):
        """Device fp64 tensors (N_blk) of S, X - S and L_new on the compact blocks."""
        import torch

        outs = [torch.empty(self.nblk_total, dtype=torch.float64, device=self.device) if w else None
                for w in (want_s, want_clean, want_l)]
        ptr = [ctypes.c_void_p(o.data_ptr()) if o is not None else ctypes.c_void_p() for o in outs]
        nat.check(self.lib.rtcur_engine_export_blocks(self.handle, *ptr))
        return outs

    def to_host(self, dev_tensors):
        """Copy fp64 device vectors into host numpy arrays the caller owns.

        Default: the arrays ARE the D2H target -- one page-locked block per call
        (torch's caching host allocator recycles it once the arrays are gone, so
        a steady stream of solves allocates nothing), filled at full PCIe rate
        and handed out as numpy views that keep it alive.  No second host copy.
        ``RTCUR_PINNED_RESULTS=0``: D2H into a staging buffer kept by the engine,
        then a multi-threaded copy into ordinary (pageable) arrays."""
        import torch

        total = sum(int(t.numel()) for t in dev_tensors)
        if PINNED_RESULTS:
            st = torch.empty(max(total, 1), dtype=torch.float64, pin_memory=True)
            o = 0
            for t in dev_tensors:
                st[o:o + t.numel()].copy_(t, non_blocking=True)
                o += t.numel()
            torch.cuda.current_stream(self.device).synchronize()
            stage = st.numpy()   # keeps ``st`` (and so the pinned block) alive through .base
            outs, o = [], 0
            for t in dev_tensors:
                outs.append(stage[o:o + int(t.numel())])
                o += int(t.numel())
            return outs
        st = getattr(self, "_pin_stage", None)
        if st is None or st.numel() < total:
            st = self._pin_stage = torch.empty(total, dtype=torch.float64, pin_memory=True)
        o = 0
        for t in dev_tensors:
            st[o:o + t.numel()].copy_(t, non_blocking=True)
            o += t.numel()
        torch.cuda.current_stream(self.device).synchronize()
        stage = st.numpy()
        outs, o = [], 0
        for t in dev_tensors:
            a = np.empty(int(t.numel()), dtype=np.float64)
            _parallel_copy(a, stage[o:o + a.size])
            outs.append(a)
            o += a.size
        return outs

    def export_cur(self):
        """Host arrays: U_k (|I|xr), sigma_k, V_k (|J|xr), A_k (d x r), G (F-order)."""
        n = self.n
        U = [np.zeros((self.row_sizes[k], self.ranks[k])) for k in range(n)]
        S = [np.zeros(self.ranks[k]) for k in range(n)]
        V = [np.zeros((self.col_sizes[k], self.ranks[k])) for k in range(n)]
        A = [np.zeros((self.ranks[k], self.shape[k])) for k in range(n)]   # col-major d x r == row-major r x d
        G = np.zeros(int(np.prod(self.ranks)))

        def arr(lst):
            return (nat.c_dp * n)(*[x.ctypes.data_as(nat.c_dp) for x in lst])

        nat.check(self.lib.rtcur_engine_export_cur(self.handle, arr(U), arr(S), arr(V), arr(A),
                                                    G.ctypes.data_as(nat.c_dp)))
        return U, S, V, [a.T.copy() for a in A], G.reshape(self.ranks, order="F")

    def full_output(self, zeta: float, want_L=True, want_S=True):
        """K3 on the bound slab: (L, S, sum (x-L-S)^2, sum x^2)."""
        import torch

        nloc = (self.slab[1] - self.slab[0]) * int(np.prod(self.shape[1:], dtype=np.int64))
        L = torch.empty(nloc, dtype=self.torch_dtype, device=self.device) if want_L else None
        S = torch.empty(nloc, dtype=self.torch_dtype, device=self.device) if (want_S and self._x is not None) else None
        nbytes = int(self.lib.rtcur_engine_full_scratch_bytes(self.handle))
        tf = torch.empty(max(nbytes // 8, 1), dtype=torch.float64, device=self.device)
        sums = (ctypes.c_double * 2)()
        nat.check(self.lib.rtcur_engine_full_output(
            self.handle, float(zeta), ctypes.c_void_p(L.data_ptr() if L is not None else 0),
            ctypes.c_void_p(S.data_ptr() if S is not None else 0), ctypes.c_void_p(tf.data_ptr()), sums))
        return L, S, float(sums[0]), float(sums[1])

    def profile(self, on: bool = True, phases=None):
        """Enable the CUDA-event phase timers; ``phases``: names to time (default all)."""
        mask = 0
        for name in phases or ():
            mask |= 1 << nat.PHASES.index(name)
        nat.check(self.lib.rtcur_engine_profile_phases(self.handle, mask))
        nat.check(self.lib.rtcur_engine_profile(self.handle, int(bool(on))))

    def profile_read(self, reset: bool = False):
        """{phase: (total_ms, launches)} of the CUDA-event phase timers."""
        k = len(nat.PHASES)
        ms = (ctypes.c_double * k)()
        cnt = (ctypes.c_int64 * k)()
        nat.check(self.lib.rtcur_engine_profile_read(self.handle, ms, cnt, k, int(bool(reset))))
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(nat.PHASES)}

    # ------------------------------------------------------------ helpers
    def split_blocks(self, flat_np):
        """Split a compact N_blk host array into (core n-d F-order, [fiber d_k x |J_k|])."""
        o = self.block_offsets
        sz = [p * q for p, q in self.block_shapes]
        core = flat_np[o[0]:o[0] + sz[0]].reshape(self.row_sizes, order="F")
        fibers = tuple(flat_np[o[k + 1]:o[k + 1] + sz[k + 1]].reshape(self.block_shapes[k + 1], order="F")
                       for k in range(self.n))
        return core, fibers
