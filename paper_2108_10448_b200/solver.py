"""RTCUR solver entry point -- drop-in for the reference's ``rtcur.solver``
(/root/reference/pkg/src/rtcur/solver.py).

Same public surface: ``SolverConfig``, ``SparseEstimate``, ``SolveResult``,
``TensorAccessor``, ``DenseTensorAccessor``, ``hard_threshold``,
``zeta_schedule``, ``sampled_relative_error``, ``rtcur``.  The iteration
order is the reference's (solver.py:1-20):

    (variant R, from the second iteration: redraw the sample)
    zeta <- gamma * zeta
    S blocks <- HT(X - L, zeta)           on the sampled blocks
    L        <- CUR assembled from X - S   (rank-r truncated intersections)
    e        <- sampled relative error of X - L - S

but every per-entry step runs on the B200 through librtcur_b200.so: the
sampled blocks live in HBM, L is evaluated in its collapsed Tucker form and
the truncated SVDs run on device.  Only the index draw (numpy PCG64, for
bit-exact sets) and scalar bookkeeping stay on the host.  There is no CPU
fallback: without the library or a CUDA device the call raises.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass
from typing import Protocol, Sequence

import numpy as np

from . import _native as nat
from .engine import marshal_sample  # noqa: E402
from .engine import Engine, acquire_engine, release_engine
from .fiber_cur import FiberCur, SampleIndices, TruncatedSvd, draw_sample_indices, sample_sizes
from .tensor import DenseTensor, DeviceTensor, as_shape

__all__ = ["SolverConfig", "SparseEstimate", "SolveResult", "TensorAccessor", "DenseTensorAccessor",
           "hard_threshold", "zeta_schedule", "sampled_relative_error", "rtcur", "RANK_DEFICIENCY_RTOL"]

RANK_DEFICIENCY_RTOL = 1e-8  # solver.py:64 (applied on device, k_svd_fin2)

# When True, rtcur() records per-phase device times (CUDA events on the solve's
# stream) into timings["device_ms"] / timings["device_launches"] (bench.py).
PROFILE = False
PROFILE_PHASES = None  # phase names timed while PROFILE (None: all)

# The reference times its phases with perf_counter around synchronous numpy
# calls (solver.py:282-356).  Here the iteration is one asynchronous device
# step, so host clocks cannot split it: with PHASE_TIMINGS (env
# RTCUR_PHASE_TIMINGS=1) every device phase is bracketed by CUDA events on the
# solve's stream and timings["gather" | "eval_lowrank" | "threshold" | "build" |
# "error"] hold device seconds (timings["timing_source"] = "device-events").
# Off (default, no event nodes in the per-iteration graphs): "build" holds the
# host-observed iteration time, the other per-phase keys 0.0
# (timings["timing_source"] = "host").
PHASE_TIMINGS = os.environ.get("RTCUR_PHASE_TIMINGS", "0") == "1"
# diagnostics: a list receives (event, iteration, perf_counter) host timestamps of the loop
_TIMELINE = None
_REF_PHASES = {"gather": ("prep", "gather"), "eval_lowrank": ("wcols",), "threshold": ("threshold",),
               "build": ("gram", "eig", "svdpost", "apass", "gpass"), "error": ("error",)}


@dataclass(frozen=True)
class SolverConfig:
    """solver.py:67-118 (same fields, defaults and validation)."""

    ranks: tuple
    eps: float = 1e-5
    zeta0: float | None = None
    gamma: float = 0.7
    upsilon: float = 3.0
    variant: str = "F"
    max_iters: int = 500
    seed: int | None = None
    row_sample_sizes: tuple | None = None
    col_sample_sizes: tuple | None = None

    def __post_init__(self):
        object.__setattr__(self, "ranks", tuple(int(r) for r in self.ranks))
        object.__setattr__(self, "variant", str(self.variant).upper())
        if len(self.ranks) == 0 or any(r < 1 for r in self.ranks):
            raise ValueError(f"ranks must be positive, got {self.ranks}")
        if not 0.0 < self.gamma < 1.0:
            raise ValueError(f"gamma must lie in (0, 1), got {self.gamma}")
        if not self.eps > 0.0:
            raise ValueError(f"eps must be positive, got {self.eps}")
        if self.zeta0 is not None and not self.zeta0 >= 0.0:
            raise ValueError(f"zeta0 must be nonnegative, got {self.zeta0}")
        if not self.upsilon > 0.0:
            raise ValueError(f"upsilon must be positive, got {self.upsilon}")
        if self.variant not in ("F", "R"):
            raise ValueError(f"variant must be 'F' or 'R', got {self.variant!r}")
        if int(self.max_iters) < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        object.__setattr__(self, "max_iters", int(self.max_iters))
        for name in ("row_sample_sizes", "col_sample_sizes"):
            v = getattr(self, name)
            if v is not None:
                object.__setattr__(self, name, tuple(int(s) for s in v))

    def resolve_sample_sizes(self, shape: Sequence[int]):
        rows, cols = sample_sizes(shape, self.ranks, self.upsilon)
        if self.row_sample_sizes is not None:
            rows = self.row_sample_sizes
        if self.col_sample_sizes is not None:
            cols = self.col_sample_sizes
        return rows, cols


class SparseEstimate:
    """Sparse-component values on the sampled positions (solver.py:121-127).

    core / fibers are copied from HBM on first access."""

    def __init__(self, loader, indices: SampleIndices, owner=None):
        self._loader = loader
        self._cache = None
        self.indices = indices
        # the FiberCur whose device state the loader reads: holding it keeps the
        # engine out of the pool (a later solve cannot overwrite these blocks)
        self._owner = owner

    def _load(self):
        if self._cache is None:
            self._cache = self._loader()
        return self._cache

    @property
    def core(self) -> np.ndarray:
        return self._load()[0]

    @property
    def fibers(self) -> tuple:
        return self._load()[1]


@dataclass(frozen=True)
class SolveResult:
    """solver.py:130-141."""

    cur: FiberCur
    sparse: SparseEstimate
    error_history: tuple
    iterations: int
    converged: bool
    diagnostics: tuple
    timings: dict
    zeta_final: float
    config: SolverConfig
    trace: tuple | None = None


class TensorAccessor(Protocol):
    """solver.py:144-159: any block source can drive a solve."""

    @property
    def shape(self) -> tuple: ...

    def core_block(self, rows) -> np.ndarray: ...

    def fiber_block(self, k: int, cols: np.ndarray) -> np.ndarray: ...

    def inf_norm(self) -> float: ...


class DenseTensorAccessor:
    """TensorAccessor over a DenseTensor (solver.py:162-192): the blocks are
    gathered on the GPU (the tensor is uploaded once)."""

    def __init__(self, t: DenseTensor):
        self._t = t
        self._dev = None

    @property
    def shape(self):
        return self._t.shape

    def device_tensor(self) -> DeviceTensor:
        if self._dev is None:
            self._dev = DeviceTensor.from_host(self._t)
        return self._dev

    def core_block(self, rows) -> np.ndarray:
        """X(I_1, ..., I_n) for 1-based sorted index sets (solver.py:170-171 ->
        tensor.py:235-240), gathered on the device as strided mode-1 fibers."""
        import torch

        shape = self.shape
        rows = [np.asarray(r, dtype=np.int64).reshape(-1) for r in rows]
        if len(rows) != len(shape):
            raise ValueError(f"{len(rows)} index sets for a {len(shape)}-mode tensor")
        for m, (r, d) in enumerate(zip(rows, shape), start=1):
            if r.size and (r.min() < 1 or r.max() > d):
                raise IndexError(f"index outside [1, {d}] for mode {m}")
        # the core block's mode-1 columns are the mode-1 fibers at (I_2, .., I_n),
        # restricted to the rows I_1: gather whole fibers, then pick the rows
        others = rows[1:]
        if others:
            grids = np.meshgrid(*others, indexing="ij")
            combo = np.zeros(grids[0].shape, dtype=np.int64)
            acc = 1
            for g, d in zip(grids, shape[1:]):
                combo += (g - 1) * acc
                acc *= d
            cols = combo.reshape(-1, order="F") + 1   # mode 2 fastest (fiber column order)
        else:
            cols = np.ones(1, dtype=np.int64)
        fib = self._gather(1, cols)                                         # d_1 x prod |I_m|
        out = fib[rows[0] - 1, :]
        return np.asfortranarray(out.reshape(tuple(r.size for r in rows), order="F"))

    def fiber_block(self, k: int, cols) -> np.ndarray:
        """C_k = X_(k)(:, J) for 1-based columns (solver.py:173-179), gathered by
        the device kernel behind the reference's ``gather_columns`` plug."""
        return self._gather(k, cols)

    def _gather(self, k: int, cols) -> np.ndarray:
        import torch

        from .tensor import fiber_base_offsets, mode_stride

        shape = self.shape
        if not 1 <= k <= len(shape):
            raise ValueError(f"mode {k} outside [1, {len(shape)}]")
        bases = fiber_base_offsets(shape, k, np.asarray(cols, dtype=np.int64).reshape(-1))
        dev = self.device_tensor()
        b = torch.from_numpy(np.ascontiguousarray(bases)).to(dev.flat.device)
        length = shape[k - 1]
        out = torch.empty(length * b.numel(), dtype=torch.float64, device=dev.flat.device)
        lib = nat.load()
        nat.check(lib.rtcur_gather_columns(dev.flat.data_ptr(), 0, dev.flat.numel(), b.data_ptr(), b.numel(),
                                           mode_stride(shape, k), length, out.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream))
        return out.cpu().numpy().reshape((length, b.numel()), order="F")

    def inf_norm(self) -> float:
        """max |x| (solver.py:182-190) by the device abs-max kernel."""
        import ctypes

        import torch

        dev = self.device_tensor()
        scratch = torch.empty(1300, dtype=torch.float64, device=dev.flat.device)
        out = ctypes.c_double()
        nat.check(nat.load().rtcur_abs_max(dev.flat.data_ptr(), 0, dev.flat.numel(), scratch.data_ptr(),
                                           ctypes.byref(out), torch.cuda.current_stream().cuda_stream))
        return float(out.value)


def hard_threshold(values, zeta: float):
    """Keep entries with |x| strictly above zeta, zero the rest (solver.py:195-199),
    evaluated by the device kernel (rtcur_hard_threshold)."""
    import torch

    if not zeta >= 0.0:
        raise ValueError(f"threshold must be nonnegative, got {zeta}")
    lib = nat.load()
    if isinstance(values, torch.Tensor):
        src = values.to(dtype=torch.float64).contiguous()
        host = None
    else:
        host = np.asarray(values, dtype=np.float64)
        src = torch.from_numpy(np.ascontiguousarray(host).reshape(-1)).cuda()
    out = torch.empty_like(src)
    nat.check(lib.rtcur_hard_threshold(src.data_ptr(), src.numel(), float(zeta), out.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream))
    if host is None:
        return out
    return out.cpu().numpy().reshape(host.shape)


def zeta_schedule(zeta0: float, gamma: float, k: int) -> float:
    """solver.py:202-206."""
    if k < 0:
        raise ValueError(f"step count must be >= 0, got {k}")
    return float(gamma) ** int(k) * float(zeta0)


def _block_norm(core, fibers) -> float:
    total = float(np.sqrt(np.sum(core * core)))
    for f in fibers:
        total += float(np.sqrt(np.sum(f * f)))
    return total


def sampled_relative_error(e_core, e_fibers, x_core, x_fibers) -> float:
    """solver.py:216-231 (host helper on given blocks)."""
    num = _block_norm(e_core, e_fibers)
    den = _block_norm(x_core, x_fibers)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / den


def _error_from_sums(e2, x2) -> float:
    """The same ratio from the device per-block sums of squares (block order:
    core, fibers 1..n, as solver.py:209-213)."""
    num = 0.0
    for v in e2:
        num += float(np.sqrt(v))
    den = 0.0
    for v in x2:
        den += float(np.sqrt(v))
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / den


class _Source:
    """Where the sampled blocks come from: a resident device tensor (gathered
    by the fused K1 gather) or a generic host TensorAccessor (blocks uploaded).

    Sharded (``slab``/``group`` given): the device tensor is this rank's mode-1
    slab of a ``global_shape`` tensor.  Every sampled entry has exactly one
    owner (the rank whose slab holds its mode-1 index): the gather fills the
    owned entries, ``shard_pack`` packs them, one all-gather of the packed
    segments (padded to the largest) moves each entry once, and ``shard_unpack``
    writes all of them into the replicated compact blocks -- bit-identical to
    an unsharded gather, so the replicated CUR build, error and stop rule run
    identically on every rank.  zeta_0 is a max all-reduce of the slab
    abs-maxima (csrc/shard_xchg.cu)."""

    def __init__(self, x, slab=None, group=None, global_shape=None):
        import torch

        self.slab = slab
        self.group = group
        self.accessor = None
        self.dev = None
        if isinstance(x, DenseTensor):
            self.dev = DeviceTensor.from_host(x)
        elif isinstance(x, DenseTensorAccessor):
            self.dev = x.device_tensor()
        elif isinstance(x, DeviceTensor):
            self.dev = x
        elif isinstance(x, torch.Tensor):
            self.dev = DeviceTensor.from_torch(x)
        elif all(hasattr(x, a) for a in ("shape", "core_block", "fiber_block", "inf_norm")):
            self.accessor = x
        else:
            raise TypeError(f"unsupported tensor source {type(x).__name__}")
        self.shape = as_shape(global_shape if global_shape is not None else
                              (self.dev.shape if self.dev is not None else x.shape))
        if slab is not None:
            lo, hi = slab
            if self.dev is None or not (0 <= lo < hi <= self.shape[0]):
                raise ValueError("a sharded solve needs a device slab [lo, hi) of mode 1")
            if tuple(self.dev.shape) != (hi - lo,) + tuple(self.shape[1:]):
                raise ValueError(f"slab tensor shape {self.dev.shape} does not match [{lo}, {hi}) of {self.shape}")

    @property
    def torch_dtype(self):
        import torch

        return self.dev.dtype if self.dev is not None else torch.float64

    def attach(self, eng: Engine):
        if self.dev is not None:
            eng.bind(self.dev.flat)
        if self.group is not None:
            import torch

            from . import dist as shard

            world = shard.group_size(self.group)
            lo_hi = shard.all_gather_host(torch.tensor(list(self.slab), dtype=torch.int64), self.group, eng.device)
            bounds = [0]
            for p in range(world):
                lo, hi = (int(v) for v in lo_hi[2 * p:2 * p + 2])
                if lo != bounds[-1]:
                    raise ValueError(f"mode-1 slabs are not contiguous in rank order (rank {p} starts at {lo})")
                bounds.append(hi)
            if bounds[-1] != self.shape[0]:
                raise ValueError(f"mode-1 slabs cover [0, {bounds[-1]}) of {self.shape[0]}")
            eng.set_shards(world, shard.group_rank(self.group), bounds)

    def reduce_max(self, v: float, device) -> float:
        if self.group is None:
            return v
        from . import dist as shard

        return shard.all_reduce_max(v, self.group, device)

    def inf_norm(self, eng: Engine) -> float:
        if self.dev is not None:
            return self.reduce_max(eng.absmax(), eng.device)
        return float(self.accessor.inf_norm())

    def load_blocks(self, eng: Engine, idx: SampleIndices):
        if self.dev is not None:
            eng.gather()
            if self.group is not None:
                from . import dist as shard

                shard.exchange_blocks(eng, self.group)
            return
        import torch

        host = np.zeros(eng.nblk_total, dtype=np.float64)
        o = eng.block_offsets
        core = np.asarray(self.accessor.core_block(idx.rows), dtype=np.float64).reshape(-1, order="F")
        host[o[0]:o[0] + core.size] = core
        for k, cols in enumerate(idx.cols, start=1):
            f = np.asarray(self.accessor.fiber_block(k, cols), dtype=np.float64).reshape(-1, order="F")
            host[o[k]:o[k] + f.size] = f
        eng.xblocks().copy_(torch.from_numpy(host), non_blocking=False)


def _make_result(eng: Engine, src: _Source, idx, cfg, history, flags, timings, zeta, converged, trace):
    import torch

    holder = {}

    def blocks():
        if "blocks" not in holder:
            s_dev, c_dev, _ = eng.export_blocks(True, True, False)
            holder["blocks"] = tuple(eng.to_host([s_dev, c_dev]))
        return holder["blocks"]

    def cur_parts():
        if "cur" not in holder:
            holder["cur"] = eng.export_cur()
        return holder["cur"]

    def load_cur(key):
        U, S, V, A, G = cur_parts()
        if key in ("core", "fibers"):
            _, c = blocks()
            core, fibers = eng.split_blocks(c)
            return {"core": DenseTensor._wrap(np.asfortranarray(core)), "fibers": fibers}
        if key == "intersections":
            return {"intersections": tuple(TruncatedSvd(u=U[k], singular_values=S[k], v=V[k])
                                           for k in range(eng.n))}
        if key == "factors":
            # F_k = C_k pinv(U_k) = A_k U~_k^T (exact identity of the collapsed form): d_k x r_k
            # times r_k x |I_k| on the host arrays the export already holds (a device matmul
            # cost three round trips, ~0.6 ms at config 1, for ~1e5 multiply-adds each)
            facs = tuple(np.ascontiguousarray(A[k] @ U[k].T) for k in range(eng.n))
            return {"factors": facs}
        if key == "tucker":
            return {"tucker": (G, tuple(A))}
        raise KeyError(key)

    def load_sparse():
        s, _ = blocks()
        return eng.split_blocks(s)

    cur = FiberCur(load_cur, idx)
    cur._engine = eng        # keep the device state alive with the result
    import weakref

    weakref.finalize(cur, release_engine, eng)   # back to the pool once the result is gone
    sparse = SparseEstimate(load_sparse, idx, owner=cur)
    return SolveResult(cur=cur, sparse=sparse, error_history=tuple(history), iterations=len(history),
                       converged=converged, diagnostics=tuple(flags), timings=timings, zeta_final=zeta,
                       config=cfg, trace=tuple(trace) if trace is not None else None)


# enqueue iteration k + 1 behind k before k's stop check (RTCUR_SPECULATE=0: one at a time)
SPECULATE = os.environ.get("RTCUR_SPECULATE", "1") != "0"


def rtcur(x, cfg: SolverConfig, record_trace: bool = False) -> SolveResult:
    """Separate a sampled observation into low-multilinear-rank + sparse
    (solver.py:260-389) on the GPU.

    x: DenseTensor (uploaded once), DeviceTensor / F-contiguous torch CUDA
    tensor (used in place, fp64 or fp32), or any TensorAccessor.
    """
    return _solve(_Source(x), cfg, record_trace)


# DRAM bytes a strided fiber element costs the gather (8-byte reads one per
# 32-byte sector, >= 64-byte DRAM fetches; ~120 B measured by ncu on config 1)
_STRIDED_BYTES = 100


_HBM_SEEN: dict = {}


def _free_hbm(device):
    """(free, total) bytes of HBM as this process can use them: the driver's figure
    (cudaMemGetInfo, refreshed at most every few seconds -- it takes a driver-wide lock
    and was seen stalling a solve's setup for milliseconds while monitoring tools poll
    the GPU) corrected by what torch's caching allocator has reserved since."""
    import torch

    key = str(device)
    now = time.monotonic()
    seen = _HBM_SEEN.get(key)
    reserved = torch.cuda.memory_reserved(device)
    if seen is None or now - seen[0] > 5.0:
        free, total = torch.cuda.mem_get_info(device)
        # memory held outside torch's allocator (other processes, contexts, the engine's own cudaMallocs)
        seen = _HBM_SEEN[key] = (now, total - free - reserved, total)
    _, other, total = seen
    cached = reserved - torch.cuda.memory_allocated(device)   # reusable without a cudaMalloc
    return total - other - reserved + cached, total


def _mode_copy_plan(shape, col_sizes, cfg, src):
    """Modes k >= 1 whose fibers the RTCUR-R gathers should read from a per-solve
    mode-k-fastest copy of X: when ~max_iters gathers of d_k |J_k| strided entries
    cost clearly more DRAM traffic than writing and reading the copy once."""
    if cfg.variant != "R" or src.dev is None or src.group is not None or len(shape) < 2:
        return ()
    import torch

    E = src.dev.flat.element_size()
    N = int(np.prod(shape, dtype=np.int64))
    gathers = min(int(cfg.max_iters), 25) + 1
    want = [k for k in range(1, len(shape))
            if gathers * shape[k] * col_sizes[k] * (_STRIDED_BYTES - E) > 1.5 * 2 * N * E]
    if not want:
        return ()
    # each copy is another N*E bytes of HBM: keep only what fits with headroom
    # (1 GiB + 10 % of the device) next to everything already allocated
    free, total = _free_hbm(src.dev.flat.device)
    room = free - (1 << 30) - total // 10
    keep = []
    for k in want:
        if room >= N * E:
            keep.append(k)
            room -= N * E
    return tuple(keep)


class _AheadSampler:
    """RTCUR-R index draws on a background thread, in stream order.

    The solve consumes the generator only through these draws (solver.py:293-317:
    the first sample, then one per iteration), so a thread that keeps drawing the
    next samples into a short queue hands the loop exactly the sets the
    reference draws, in the same order.  The draw itself runs in native code
    without the GIL (rtcur_draw_distinct), so it overlaps the loop's own host
    work (staging, launches, the stop check) instead of adding to it: at config 1
    the host loop was ~60 % draw and paced the device.  Draws past the last
    iteration are discarded (the generator is local to the solve)."""

    def __init__(self, shape, row_sizes, col_sizes, rng, depth: int = 3):
        import queue
        import threading

        self._args = (shape, row_sizes, col_sizes, rng)
        self.views = {}   # id(sample) -> its marshalled view, taken by the loop's set_sample
        self._q = queue.Queue(maxsize=depth)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, name="rtcur-sampler", daemon=True)
        self._t.start()

    def _run(self):
        import queue

        shape, row_sizes, col_sizes, rng = self._args
        while not self._stop.is_set():
            try:
                item = draw_sample_indices(shape, row_sizes, col_sizes, rng)
                self.views[id(item)] = marshal_sample(item)   # the C-ABI view, off the loop's thread
            except BaseException as exc:   # surfaced by next()
                item = exc
            while not self._stop.is_set():
                try:
                    self._q.put(item, timeout=0.05)
                    break
                except queue.Full:
                    continue
            if isinstance(item, BaseException):
                return

    def next(self):
        item = self._q.get()
        if isinstance(item, BaseException):
            raise item
        return item

    def close(self):
        import queue

        self._stop.set()
        try:
            while True:
                self._q.get_nowait()
        except queue.Empty:
            pass
        self._t.join()


def _solve(src: "_Source", cfg: SolverConfig, record_trace: bool = False, on_iteration=None) -> SolveResult:
    """The solve loop.  ``on_iteration(k, eng, idx, zeta, err, flags)`` (optional,
    parity tooling) runs after every iteration, while the engine still holds
    that iteration's state (``eng.export_blocks`` / ``eng.export_cur``)."""
    import torch

    shape = src.shape
    if len(cfg.ranks) != len(shape):
        raise ValueError(f"{len(cfg.ranks)} ranks for a {len(shape)}-mode tensor")
    for m, (r, d) in enumerate(zip(cfg.ranks, shape), start=1):
        if r > d:
            raise ValueError(f"mode {m}: rank {r} exceeds extent {d}")
    timings = {k: 0.0 for k in ("sample", "gather", "eval_lowrank", "threshold", "build", "error", "total")}
    t_start = time.perf_counter()
    rng = np.random.default_rng(cfg.seed)
    row_sizes, col_sizes = cfg.resolve_sample_sizes(shape)

    for m, (r, rs, cs) in enumerate(zip(cfg.ranks, row_sizes, col_sizes), start=1):
        if r > rs or r > cs:   # fiber_cur.py:257-261 (raised before any work, as there)
            raise ValueError(f"mode {m}: rank {r} exceeds sample sizes (|rows|={rs}, |cols|={cs})")

    if _TIMELINE is not None:
        _TIMELINE.append(("enter", 0, time.perf_counter()))
    eng = acquire_engine(shape, cfg.ranks, row_sizes, col_sizes, src.torch_dtype, slab=src.slab)
    if _TIMELINE is not None:
        _TIMELINE.append(("engine", 0, time.perf_counter()))
    phase_events = PHASE_TIMINGS and not PROFILE
    if PROFILE:
        eng.profile(True, PROFILE_PHASES)
    elif phase_events:
        eng.profile(True, None)
        eng.profile_read(reset=True)
    eng.reset()
    src.attach(eng)
    copies = _mode_copy_plan(shape, col_sizes, cfg, src)
    if copies:
        eng.bind_mode_copies(src.dev.flat, copies)
    if _TIMELINE is not None:
        _TIMELINE.append(("copies", 0, time.perf_counter()))
    sampler = None
    try:
        # the device scans max|X| (and builds the mode copies) while the host draws the
        # first sample (the generator is consumed by sampling only, solver.py:293-316)
        early_zeta = (cfg.zeta0 is None and src.dev is not None
                      and os.environ.get("RTCUR_EARLY_ZETA", "1") != "0")
        if early_zeta:
            eng.absmax_begin()
        # RTCUR-R: every draw (the first one included) from the background sampler
        sampler = (_AheadSampler(shape, row_sizes, col_sizes, rng)
                   if cfg.variant == "R" and cfg.max_iters > 1 and os.environ.get("RTCUR_AHEAD_SAMPLER", "1") != "0"
                   else None)
        draw = sampler.next if sampler is not None else (lambda: draw_sample_indices(shape, row_sizes, col_sizes, rng))
        views = sampler.views if sampler is not None else {}
        t0 = time.perf_counter()
        idx = draw()
        timings["sample"] += time.perf_counter() - t0
        if _TIMELINE is not None:
            _TIMELINE.append(("first_draw", 0, time.perf_counter()))
        t0 = time.perf_counter()
        eng.set_sample(idx, views.pop(id(idx), None))
        src.load_blocks(eng, idx)
        timings["gather"] += time.perf_counter() - t0

        if _TIMELINE is not None:
            _TIMELINE.append(("staged0", 0, time.perf_counter()))
        if cfg.zeta0 is not None:
            zeta = float(cfg.zeta0)
        else:
            zeta = src.reduce_max(eng.absmax_end(), eng.device) if early_zeta else src.inf_norm(eng)
        if _TIMELINE is not None:
            _TIMELINE.append(("zeta0", 0, time.perf_counter()))
        t_loop = time.perf_counter()
        history, flags = [], []
        trace = [] if record_trace else None
        converged = False
        # RTCUR-R draws the next sample while the GPU runs the current iteration:
        # the generator is consumed by sampling only, so drawing ahead leaves every
        # index set identical to the reference's (solver.py:315-317).
        # device-resident local tensors: the next sample's upload and gather go into the
        # engine's inactive sample slot right behind the running iteration (no host gap)
        prefetch = src.dev is not None
        # Speculation: iteration k + 1 is enqueued while k is still running, so the stream
        # never idles over the host's stop check (solver.py:357-358); the device evaluates
        # the same test at the end of k and k + 1's kernels return at once when it
        # holds.  Needs the engine's state untouched between iterations: not with a
        # trace / iteration callback, a host accessor or a sharded exchange.
        eng.set_eps(cfg.eps)
        spec = (SPECULATE and src.dev is not None and src.group is None and not record_trace
                and on_iteration is None and eng.can_speculate())
        resample = cfg.variant == "R"

        def stage(sample):
            # upload + gather into a free sample slot of the engine (on its side stream when an
            # iteration is in flight: under that iteration's eigensolver)
            t1 = time.perf_counter()
            eng.set_sample(sample, views.pop(id(sample), None))
            src.load_blocks(eng, sample)
            timings["gather"] += time.perf_counter() - t1

        def draw_next():
            t1 = time.perf_counter()
            smp = draw()
            timings["sample"] += time.perf_counter() - t1
            return smp

        k = 1
        zeta *= cfg.gamma
        t0 = time.perf_counter()
        if _TIMELINE is not None:
            _TIMELINE.append(("async", k, t0))
        eng.iterate_async(zeta, first=True)
        nxt, nxt_staged = None, False   # RTCUR-R: the sample of iteration k + 1, once drawn / staged
        while True:
            # iteration k is in flight with sample `idx` at threshold `zeta`
            ahead, launched = False, None
            more = k < cfg.max_iters
            if resample and more and nxt is None:
                nxt = draw_next()
                if prefetch:
                    stage(nxt)
                    nxt_staged = True
            if spec and more and (nxt_staged or not resample):
                eng.iterate_async(zeta * cfg.gamma, first=False)
                ahead, launched = True, nxt
                nxt, nxt_staged = None, False
                # the sample after next goes to the third slot while k and k + 1 run, so the
                # host's staging work is off the path between k's result and k + 2's launch
                if resample and k + 1 < cfg.max_iters:
                    nxt = draw_next()
                    stage(nxt)
                    nxt_staged = True
            if _TIMELINE is not None:
                _TIMELINE.append(("staged", k, time.perf_counter()))
            e2, x2, fl = eng.iterate_wait()
            timings["build"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            if _TIMELINE is not None:
                _TIMELINE.append(("waited", k, t0))
            err = _error_from_sums(e2, x2)
            history.append(err)
            flags.append(fl)
            stop = err <= cfg.eps
            if ahead and stop != eng.last_stop():
                raise RuntimeError(f"device stop rule disagrees with the host at iteration {k} (err {err!r})")
            if record_trace:
                s_dev, _, l_dev = eng.export_blocks(True, False, True)
                s_core, s_fib = eng.split_blocks(s_dev.cpu().numpy())
                l_core, l_fib = eng.split_blocks(l_dev.cpu().numpy())
                trace.append({"iteration": k, "zeta": zeta, "indices": idx, "s_core": s_core, "s_fibers": s_fib,
                              "l_core": l_core, "l_fibers": l_fib, "error": err})
            if on_iteration is not None:
                on_iteration(k, eng, idx, zeta, err, fl)
            if stop:
                converged = True
                if ahead:
                    eng.iterate_cancel()   # k + 1 ran nothing: k stays the engine's iterate
                break
            if k >= cfg.max_iters:
                break
            k += 1
            zeta *= cfg.gamma
            if ahead:
                if resample:
                    idx = launched
            else:
                if resample:
                    idx = nxt
                    if not nxt_staged:
                        stage(idx)
                    nxt, nxt_staged = None, False
                if _TIMELINE is not None:
                    _TIMELINE.append(("async", k, time.perf_counter()))
                eng.iterate_async(zeta, first=False)
    finally:
        if sampler is not None:
            sampler.close()
        if copies:
            eng.bind_mode_copies(None, ())   # the loop is done (or failed); exports do not gather
    timings["loop"] = time.perf_counter() - t_loop
    timings["total"] = time.perf_counter() - t_start
    timings["timing_source"] = "host"
    if PROFILE or phase_events:
        ph = eng.profile_read(reset=True)
        if PROFILE:
            timings["device_ms"] = {k: v[0] for k, v in ph.items()}
            timings["device_launches"] = {k: v[1] for k, v in ph.items()}
        if PROFILE_PHASES is None:   # every phase timed: the reference's keys from device events
            timings["host_loop"] = timings["build"]
            for key, names in _REF_PHASES.items():
                timings[key] = 1e-3 * sum(ph[nm][0] for nm in names)
            timings["timing_source"] = "device-events"
        eng.profile(False)
    return _make_result(eng, src, idx, cfg, history, flags, timings, zeta, converged, trace)
