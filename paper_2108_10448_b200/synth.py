"""Seeded synthetic RTCUR instances with the BASELINE.json config shapes.

BASELINE names no public dataset; every config is a
seeded synthetic stand-in.  Host generation is numpy (PCG64) so the CPU oracle
and the GPU path see byte-identical X; the reference's own generator
(/root/reference/pkg/src/rtcur/synth.py:74-130, exact-count outliers, c=1) is
deliberately NOT used because BASELINE specifies Bernoulli(alpha) support with
c=10.

Layout contract (tensor.py:1-10 of the reference): mode-1-fastest ("F"-order)
flat buffer.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["BaselineConfig", "CONFIGS", "make_gaussian_tucker", "make_video_like", "make_config",
           "baseline_sample_sizes", "InstanceSpec", "gen_lowrank_device", "gen_outliers_device",
           "make_instance_device", "make_gaussian_tucker_device", "make_config_device", "slab_bounds"]


@dataclass(frozen=True)
class BaselineConfig:
    index: int
    variant: str
    shape: tuple
    ranks: tuple
    alpha: float
    c: float
    eps: float
    dtype: str  # "f64" | "f32"
    kind: str = "gaussian"  # "gaussian" | "video"

    @property
    def seed_instance(self) -> int:
        return 1000 + self.index

    @property
    def seed_solver(self) -> int:
        return self.index


CONFIGS = {
    0: BaselineConfig(0, "F", (100, 100, 100), (3, 3, 3), 0.2, 10.0, 1e-5, "f64"),
    1: BaselineConfig(1, "R", (400, 400, 400), (5, 5, 5), 0.3, 10.0, 1e-5, "f64"),
    2: BaselineConfig(2, "F", (1200, 1200, 1200), (10, 10, 10), 0.2, 10.0, 1e-5, "f32"),
    3: BaselineConfig(3, "F", (240, 320, 3, 600), (10, 10, 3, 2), 0.0, 1.0, 1e-4, "f32", "video"),
    4: BaselineConfig(4, "R", (220, 220, 220, 220), (4, 4, 4, 4), 0.2, 10.0, 1e-5, "f32"),
}


def baseline_sample_sizes(shape, ranks):
    """BASELINE |I_i| = ceil(3 r ln d) (clamped to d), |J_i| = ceil(3 r^2 ln^2 d).

    Passed through SolverConfig.row_sample_sizes / col_sample_sizes, the
    reference's own override (solver.py:110-118).
    """
    rows = tuple(min(d, max(1, math.ceil(3 * r * math.log(d)))) for d, r in zip(shape, ranks))
    total = int(np.prod(shape, dtype=np.int64))
    cols = tuple(min(total // d, math.ceil(3 * r * r * math.log(d) ** 2)) for d, r in zip(shape, ranks))
    return rows, cols


def _tucker(core: np.ndarray, factors) -> np.ndarray:
    """core x_1 Y_1 ... x_n Y_n on F-ordered arrays, returns F-ordered array."""
    out = core
    for k, y in enumerate(factors):
        shp = out.shape
        unf = np.reshape(np.moveaxis(out, k, 0), (shp[k], -1), order="F")
        prod = y @ unf
        rest = tuple(d for j, d in enumerate(shp) if j != k)
        out = np.moveaxis(prod.reshape((y.shape[0],) + rest, order="F"), 0, k)
    return np.asfortranarray(out)


def make_gaussian_tucker(shape, ranks, alpha, c, seed, dtype=np.float64):
    """L* = G x_i Y_i (all iid N(0,1)); S* Bernoulli(alpha) support, values
    iid U[-c mean|L*|, c mean|L*|]; X = L* + S*.  Returns flat F-order
    (x, l_star, s_star) in ``dtype`` (fp32 configs round the fp64 draw)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(int(np.prod(ranks))).reshape(ranks, order="F")
    ys = [rng.standard_normal((d, r)) for d, r in zip(shape, ranks)]
    low = _tucker(g, ys).reshape(-1, order="F")
    mu = float(np.mean(np.abs(low)))
    mask = rng.random(low.size) < alpha
    sp = np.zeros(low.size)
    sp[mask] = rng.uniform(-c * mu, c * mu, size=int(mask.sum()))
    x = low + sp
    return x.astype(dtype), low.astype(dtype), sp.astype(dtype)


def make_video_like(shape=(240, 320, 3, 600), ranks=(10, 10, 3, 2), n_blocks=40, block=16, seed=1003,
                    dtype=np.float32):
    """Config-3 stand-in: H x W x C x T background of multilinear rank
    (10,10,3,2) = Gaussian core x orthonormalised Gaussian factors, scaled
    rank-preservingly by 1/max|L| (an affine map to [0,1] would add a constant
    and raise the rank); foreground = ``n_blocks`` axis-aligned 16x16 blocks
    moving with constant random velocity (bouncing at the borders), iid
    U[0,1] values on all colour channels (same support per channel)."""
    rng = np.random.default_rng(seed)
    h, w, ch, t = shape
    g = rng.standard_normal(int(np.prod(ranks))).reshape(ranks, order="F")
    qs = []
    for d, r in zip(shape, ranks):
        q, _ = np.linalg.qr(rng.standard_normal((d, r)))
        qs.append(q)
    low = _tucker(g, qs)
    low /= float(np.max(np.abs(low)))
    sp = np.zeros(shape, order="F")
    pos = np.stack([rng.uniform(0, h - block, n_blocks), rng.uniform(0, w - block, n_blocks)], 1)
    vel = rng.uniform(-3.0, 3.0, (n_blocks, 2))
    for f in range(t):
        for b in range(n_blocks):
            r0, c0 = int(pos[b, 0]), int(pos[b, 1])
            vals = rng.random((block, block, ch))
            sp[r0:r0 + block, c0:c0 + block, :, f] = vals
        pos += vel
        for ax, lim in ((0, h - block), (1, w - block)):
            lo = pos[:, ax] < 0
            hi = pos[:, ax] > lim
            vel[lo | hi, ax] *= -1.0
            pos[:, ax] = np.clip(pos[:, ax], 0, lim)
    x = (low + sp).reshape(-1, order="F")
    return x.astype(dtype), low.reshape(-1, order="F").astype(dtype), sp.reshape(-1, order="F").astype(dtype)


def make_config(index: int):
    """(x_flat, l_star_flat, s_star_flat, cfg) for BASELINE config ``index``."""
    cfg = CONFIGS[index]
    dt = np.float64 if cfg.dtype == "f64" else np.float32
    if cfg.kind == "video":
        x, low, sp = make_video_like(cfg.shape, cfg.ranks, seed=cfg.seed_instance, dtype=dt)
    else:
        x, low, sp = make_gaussian_tucker(cfg.shape, cfg.ranks, cfg.alpha, cfg.c, cfg.seed_instance, dt)
    return x, low, sp, cfg


# ----------------------------------------------------------------- device generation (configs 2-4)


def slab_bounds(d1: int, world: int, rank: int):
    """Mode-1 slab of `rank` among `world` (contiguous, sizes differ by at most 1;
    220/8 -> 28/27 rows)."""
    return (d1 * rank) // world, (d1 * (rank + 1)) // world


def make_gaussian_tucker_device(shape, ranks, alpha, c, seed, dtype=None, slab=None, group=None, mu=None):
    """Device-side instance with the same law as ``make_gaussian_tucker``:
    L* = G x_i Y_i (iid N(0,1) core and factors, drawn on the host from
    ``seed``), S* Bernoulli(alpha) with values U[-c mean|L*|, c mean|L*|] keyed
    by (seed, global element index).  Every entry is bitwise independent of the
    slab decomposition (the mode>=2 contraction Tf is shared; the mode-1 step is
    a fixed-order per-entry dot product in ``rtcur_generate_tucker``).  Returns
    this rank's mode-1 slab as a DeviceTensor (shape (hi-lo, d_2, ..)) and
    mean|L*| (all-reduced over ``group``, or taken from ``mu``)."""
    import torch

    from . import _native as nat
    from .tensor import DeviceTensor

    dtype = dtype or torch.float32
    n = len(shape)
    lo, hi = slab or (0, shape[0])
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(int(np.prod(ranks))).reshape(ranks, order="F")
    ys = [rng.standard_normal((d, r)) for d, r in zip(shape, ranks)]
    dev = torch.device("cuda", torch.cuda.current_device())
    r1 = ranks[0]
    # Tf[R, a] = (G x_{m>=2} Y_m)[a, i_2, .., i_n], R = i_2 + d_2 i_3 + ... (host, exact same bits on every rank)
    tf = g
    for m in range(1, n):
        tf = np.tensordot(tf, ys[m], axes=([1], [1]))   # contract the next rank axis, append the mode axis
    tf = np.moveaxis(tf, 0, -1)                          # (i_2, .., i_n, a)
    tf = np.ascontiguousarray(np.transpose(tf, tuple(range(n - 2, -1, -1)) + (n - 1,)) if n > 1 else tf)
    Tf = torch.from_numpy(tf.reshape(-1, r1)).to(dev)
    Y1 = torch.from_numpy(np.asfortranarray(ys[0]).reshape(-1, order="F")).to(dev)
    ncols = int(np.prod(shape[1:], dtype=np.int64)) if n > 1 else 1
    lib = nat.load()
    scratch = torch.empty(1300, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    dt_code = 0 if dtype == torch.float64 else 1
    if mu is None:
        import ctypes

        s_abs = ctypes.c_double()
        nat.check(lib.rtcur_generate_tucker(Y1.data_ptr(), Tf.data_ptr(), shape[0], r1, lo, hi, ncols, 0, int(seed),
                                            float(alpha), 0.0, dt_code, None, scratch.data_ptr(),
                                            ctypes.byref(s_abs), stream))
        tot = torch.tensor([s_abs.value], dtype=torch.float64, device=dev)
        if group is not None:
            import torch.distributed as dist

            if dist.get_backend(group) != "nccl":   # gloo groups reduce host tensors
                tot = tot.cpu()
            dist.all_reduce(tot, group=group)
        mu = float(tot.item()) / float(np.prod(shape, dtype=np.float64))
    X = torch.empty((hi - lo) * ncols, dtype=dtype, device=dev)
    nat.check(lib.rtcur_generate_tucker(Y1.data_ptr(), Tf.data_ptr(), shape[0], r1, lo, hi, ncols, 1, int(seed),
                                        float(alpha), float(c * mu), dt_code, X.data_ptr(), scratch.data_ptr(), None,
                                        stream))
    return DeviceTensor(X, (hi - lo,) + tuple(shape[1:])), mu


def make_config_device(index: int, slab=None, group=None):
    """BASELINE config ``index`` generated on the GPU (slab of mode 1 when sharded)."""
    import torch

    cfg = CONFIGS[index]
    dt = torch.float64 if cfg.dtype == "f64" else torch.float32
    if cfg.kind == "video":
        from .tensor import DeviceTensor

        x, _, _ = make_video_like(cfg.shape, cfg.ranks, seed=cfg.seed_instance, dtype=np.float32)
        lo, hi = slab or (0, cfg.shape[0])
        full = torch.from_numpy(x).cuda().reshape(tuple(reversed(cfg.shape)))
        part = full[..., lo:hi].contiguous() if slab else full
        return DeviceTensor(part.reshape(-1), (hi - lo,) + tuple(cfg.shape[1:])), cfg
    X, _ = make_gaussian_tucker_device(cfg.shape, cfg.ranks, cfg.alpha, cfg.c, cfg.seed_instance, dt, slab, group)
    return X, cfg


# ----------------------------------------------------------------- reference generator semantics on the device


@dataclass(frozen=True)
class InstanceSpec:
    """Mirror of the reference's InstanceSpec (synth.py:41-72): a d x ... x d tensor
    of order n, multilinear rank (r, ..., r), outlier fraction alpha."""

    n: int
    d: int
    r: int
    alpha: float
    seed: int

    def __post_init__(self):
        if int(self.n) < 1:
            raise ValueError(f"order must be >= 1, got {self.n}")
        if int(self.d) < 1:
            raise ValueError(f"extent must be >= 1, got {self.d}")
        if not 1 <= int(self.r) <= int(self.d):
            raise ValueError(f"rank {self.r} outside [1, {self.d}]")
        if not 0.0 <= float(self.alpha) < 1.0:
            raise ValueError(f"outlier fraction must lie in [0, 1), got {self.alpha}")
        object.__setattr__(self, "n", int(self.n))
        object.__setattr__(self, "d", int(self.d))
        object.__setattr__(self, "r", int(self.r))
        object.__setattr__(self, "alpha", float(self.alpha))

    @property
    def shape(self) -> tuple:
        return (self.d,) * self.n

    @property
    def ranks(self) -> tuple:
        return (self.r,) * self.n


def _tucker_device(core: np.ndarray, ys, dtype=None):
    """L = core x_1 Y_1 ... x_n Y_n on the device (rtcur_generate_tucker with no
    outliers): Tf = core x_{m>=2} Y_m on the host (small), the mode-1 step and
    the |L| sum on the device.  Returns (flat torch tensor, sum |L|)."""
    import ctypes

    import torch

    from . import _native as nat

    dtype = dtype or torch.float64
    n = len(ys)
    shape = tuple(int(y.shape[0]) for y in ys)
    r1 = int(ys[0].shape[1])
    tf = core
    for m in range(1, n):
        tf = np.tensordot(tf, ys[m], axes=([1], [1]))
    tf = np.moveaxis(tf, 0, -1)
    tf = np.ascontiguousarray(np.transpose(tf, tuple(range(n - 2, -1, -1)) + (n - 1,)) if n > 1 else tf)
    dev = torch.device("cuda", torch.cuda.current_device())
    Tf = torch.from_numpy(tf.reshape(-1, r1)).to(dev)
    Y1 = torch.from_numpy(np.asfortranarray(ys[0]).reshape(-1, order="F")).to(dev)
    ncols = int(np.prod(shape[1:], dtype=np.int64)) if n > 1 else 1
    lib = nat.load()
    scratch = torch.empty(1300, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    dt = 0 if dtype == torch.float64 else 1
    s_abs = ctypes.c_double()
    nat.check(lib.rtcur_generate_tucker(Y1.data_ptr(), Tf.data_ptr(), shape[0], r1, 0, shape[0], ncols, 0, 0, 0.0, 0.0,
                                        dt, None, scratch.data_ptr(), ctypes.byref(s_abs), stream))
    L = torch.empty(shape[0] * ncols, dtype=dtype, device=dev)
    nat.check(lib.rtcur_generate_tucker(Y1.data_ptr(), Tf.data_ptr(), shape[0], r1, 0, shape[0], ncols, 1, 0, 0.0, 0.0,
                                        dt, L.data_ptr(), scratch.data_ptr(), None, stream))
    return L, float(s_abs.value)


def gen_lowrank_device(spec: InstanceSpec):
    """synth.py:74-88 on the device: the same core/factor draws (host PCG64,
    core first, then the factors mode by mode), the expansion in HBM.
    Returns an fp64 DeviceTensor."""
    from .tensor import DeviceTensor

    rng = np.random.default_rng(spec.seed)
    core = rng.standard_normal(spec.r ** spec.n).reshape((spec.r,) * spec.n, order="F")
    ys = [rng.standard_normal((spec.d, spec.r)) for _ in range(spec.n)]
    L, _ = _tucker_device(core, ys)
    return DeviceTensor(L, spec.shape)


def gen_outliers_device(low, alpha: float, seed, x=None):
    """synth.py:101-121 on the device: floor(alpha * size) positions drawn
    without replacement by the reference's sampler (same generator stream),
    values uniform on [-mu, mu] with mu = mean|low| (fixed-order device sum).
    Returns the sparse DeviceTensor; when ``x`` (a copy of low) is given it is
    updated in place to low + sparse."""
    import ctypes

    import torch

    from . import _native as nat
    from .fiber_cur import _draw_without_replacement
    from .tensor import DeviceTensor

    if not 0.0 <= alpha < 1.0:
        raise ValueError(f"outlier fraction must lie in [0, 1), got {alpha}")
    size = int(low.flat.numel())
    count = int(math.floor(alpha * size + 1e-9))
    S = torch.zeros(size, dtype=torch.float64, device=low.flat.device)
    if count > 0:
        rng = np.random.default_rng(seed)
        pos = _draw_without_replacement(rng, size, count) - 1
        lf = low.flat if low.flat.dtype == torch.float64 else low.flat.double()
        scratch = torch.empty(600, dtype=torch.float64, device=lf.device)
        tot = ctypes.c_double()
        nat.check(nat.load().rtcur_abs_sum(lf.data_ptr(), size, scratch.data_ptr(), ctypes.byref(tot),
                                           torch.cuda.current_stream().cuda_stream))
        mu = tot.value / size
        u = rng.random(count)
        dev = low.flat.device
        pos_d = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.int64)).to(dev)
        u_d = torch.from_numpy(u).to(dev)
        target = x.flat if x is not None else torch.zeros(size, dtype=torch.float64, device=dev)
        nat.check(nat.load().rtcur_scatter_outliers(target.data_ptr(), pos_d.data_ptr(), u_d.data_ptr(), count,
                                                    ctypes.c_double(mu), S.data_ptr(),
                                                    torch.cuda.current_stream().cuda_stream))
    return DeviceTensor(S, low.shape)


def make_instance_device(spec: InstanceSpec):
    """synth.py:124-135 on the device: (x, low, sparse) fp64 DeviceTensors; the
    outlier stream is seeded by SeedSequence([seed, 1]) as in the reference."""
    from .tensor import DeviceTensor

    low = gen_lowrank_device(spec)
    x = DeviceTensor(low.flat.clone(), low.shape)
    sparse = gen_outliers_device(low, spec.alpha, np.random.SeedSequence([spec.seed, 1]), x=x)
    return x, low, sparse
