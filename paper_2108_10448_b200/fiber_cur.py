"""Fiber-CUR sample and result containers (mirror of the reference's
``rtcur.fiber_cur`` / ``rtcur.linalg`` public types,
/root/reference/pkg/src/rtcur/fiber_cur.py and linalg.py).

Index sampling stays on the host and consumes ``np.random.default_rng`` in
exactly the reference's order (fiber_cur.py:148-209), so index sets are
bit-identical to the reference's for equal seeds (same numpy build).
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .tensor import DenseTensor, as_shape

__all__ = ["SampleIndices", "FiberCur", "TruncatedSvd", "sample_sizes", "sample_indices", "draw_sample_indices",
           "PINV_RTOL"]

PINV_RTOL = 1e-12  # linalg.py:23


@dataclass(frozen=True)
class SampleIndices:
    """Per-mode 1-based sorted index sets (fiber_cur.py:50-83)."""

    rows: tuple
    cols: tuple

    def row_sizes(self) -> tuple[int, ...]:
        return tuple(int(r.size) for r in self.rows)

    def col_sizes(self) -> tuple[int, ...]:
        return tuple(int(c.size) for c in self.cols)

    def validate_for(self, shape: Sequence[int]) -> None:
        shape = as_shape(shape)
        n = len(shape)
        if len(self.rows) != n or len(self.cols) != n:
            raise ValueError(f"sample has {len(self.rows)} row sets / {len(self.cols)} column sets "
                             f"for a {n}-mode tensor")
        total = int(np.prod(shape, dtype=np.int64))
        for m, (r, c, d) in enumerate(zip(self.rows, self.cols, shape), start=1):
            if r.size == 0 or c.size == 0:
                raise ValueError(f"mode {m}: empty sample set")
            if r[0] < 1 or r[-1] > d:
                raise IndexError(f"mode {m}: row index outside [1, {d}]")
            rest = total // d
            if c[0] < 1 or c[-1] > rest:
                raise IndexError(f"mode {m}: fiber column outside [1, {rest}]")


@dataclass(frozen=True)
class TruncatedSvd:
    """Rank-r factorisation M_r = u diag(s) v^T (linalg.py:26-56)."""

    u: np.ndarray
    singular_values: np.ndarray
    v: np.ndarray

    @property
    def rank(self) -> int:
        return int(self.singular_values.size)

    def reconstruct(self) -> np.ndarray:
        return (self.u * self.singular_values) @ self.v.T

    def pinv(self) -> np.ndarray:
        s = self.singular_values
        tau = max(self.u.shape[0], self.v.shape[0]) * float(s[0]) * PINV_RTOL
        inv = np.divide(1.0, s, out=np.zeros_like(s), where=s > tau)
        return (self.v * inv) @ self.u.T


class FiberCur:
    """Sampled CUR decomposition (fiber_cur.py:86-107).

    core / fibers / intersections / factors are materialised from HBM on first
    access (the solve itself never needs them on the host); ``tucker`` gives
    the exact device-side collapsed form (G, A_1..A_n) with
    core x_i factors[i] == G x_i A_i.
    """

    def __init__(self, loader, indices: SampleIndices):
        self._loader = loader
        self._cache = {}
        self.indices = indices

    def _get(self, key):
        if key not in self._cache:
            self._cache.update(self._loader(key))
        return self._cache[key]

    @property
    def core(self) -> DenseTensor:
        return self._get("core")

    @property
    def fibers(self) -> tuple:
        return self._get("fibers")

    @property
    def intersections(self) -> tuple:
        return self._get("intersections")

    @property
    def factors(self) -> tuple:
        return self._get("factors")

    @property
    def tucker(self):
        """(G, (A_1, ..., A_n)) host arrays: G is r_1 x ... x r_n (F-order), A_k is d_k x r_k."""
        return self._get("tucker")

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(int(a.shape[0]) for a in self.tucker[1])

    def __repr__(self) -> str:
        return f"FiberCur(rows={self.indices.row_sizes()}, cols={self.indices.col_sizes()})"


def _check_ranks(shape, ranks):
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != len(shape):
        raise ValueError(f"{len(ranks)} ranks for a {len(shape)}-mode tensor")
    for m, (r, d) in enumerate(zip(ranks, shape), start=1):
        if r < 1:
            raise ValueError(f"mode {m}: rank must be >= 1, got {r}")
        if r > d:
            raise ValueError(f"mode {m}: rank {r} exceeds extent {d}")
    return ranks


def sample_sizes(shape: Sequence[int], ranks: Sequence[int], upsilon: float):
    """fiber_cur.py:110-130: |I_i| = min(d, max(r, ceil(ups r ln d))), |J_i| likewise over prod_{j!=i} d_j."""
    shape = as_shape(shape)
    ranks = _check_ranks(shape, ranks)
    if not upsilon > 0:
        raise ValueError(f"sampling constant must be positive, got {upsilon}")
    total = int(np.prod(shape, dtype=np.int64))
    rows, cols = [], []
    for d, r in zip(shape, ranks):
        rest = total // d
        rows.append(min(d, max(r, math.ceil(upsilon * r * math.log(d)))))
        cols.append(min(rest, max(r, math.ceil(upsilon * r * math.log(rest)))))
    return tuple(rows), tuple(cols)


_SEEN = threading.local()


def _seen_mask(population: int) -> np.ndarray:
    """Per-thread zeroed membership mask, reused across draws (the draw clears
    exactly the entries it set, so a 10^7-entry population is not re-zeroed on
    every RTCUR-R iteration)."""
    cache = getattr(_SEEN, "masks", None)
    if cache is None:
        cache = _SEEN.masks = {}
    m = cache.get(population)
    if m is None:
        m = cache[population] = np.zeros(population, dtype=np.uint8)
    return m


def _bitgen_iface(rng: np.random.Generator):
    """(state address, next_uint32 function address) of the generator's bit
    generator (numpy's documented ctypes interface; numpy caches it)."""
    import ctypes

    c = rng.bit_generator.ctypes
    return c.state_address, ctypes.cast(c.next_uint32, ctypes.c_void_p).value


def _seen_bits(population: int) -> np.ndarray:
    """Per-thread zeroed membership bitmap (uint64 words), reused across draws."""
    cache = getattr(_SEEN, "bits", None)
    if cache is None:
        cache = _SEEN.bits = {}
    m = cache.get(population)
    if m is None:
        m = cache[population] = np.zeros((population + 63) // 64, dtype=np.uint64)
    return m


def _draw_without_replacement(rng: np.random.Generator, population: int, k: int) -> np.ndarray:
    """fiber_cur.py:189-209 (permutation for 3k >= pop, else iid stream + first-unique)."""
    if k >= population:
        return np.arange(1, population + 1, dtype=np.int64)
    if 3 * k >= population:
        picked = rng.permutation(population)[:k]
        return np.sort(picked.astype(np.int64)) + 1
    # Same generator calls as the reference (so the same stream); the
    # first-occurrence dedup of np.unique(..., return_index=True) is done in
    # O(n) by the native helper.
    from . import _native

    lib = _native.load()
    if population <= 0xFFFFFFFF:
        # the whole draw natively on numpy's own bit generator (rtcur_draw_distinct:
        # numpy's bounded-integer algorithm on next_uint32, identical stream)
        state, nxt = _bitgen_iface(rng)
        bits = _seen_bits(population)
        out = np.empty(3 * k + 32, dtype=np.int64)
        with rng.bit_generator.lock:
            got = int(lib.rtcur_draw_distinct(state, nxt, population, k, bits.ctypes.data, out.ctypes.data,
                                              out.size))
        if got != k:
            raise RuntimeError(f"rtcur_draw_distinct failed ({got})")
        return out[:k].copy()
    seen = _seen_mask(population)
    cap = 2 * k + 64
    out = np.empty(cap, dtype=np.int64)
    nout = 0
    while nout < k:
        need = k - nout
        batch = rng.integers(0, population, size=need + need // 2 + 16, dtype=np.int64)
        if nout + batch.size > out.size:
            out = np.concatenate([out, np.empty(nout + batch.size, dtype=np.int64)])
        got = int(lib.rtcur_append_distinct(out.ctypes.data, nout, batch.ctypes.data, batch.size, seen.ctypes.data,
                                            population))
        if got < 0:
            seen[:] = 0
            raise RuntimeError("rtcur_append_distinct: index outside the population")
        nout = got
    seen[out[:nout]] = 0
    return np.sort(out[:k]) + 1


def draw_sample_indices(shape, row_sizes, col_sizes, rng: np.random.Generator) -> SampleIndices:
    """fiber_cur.py:148-174: row sets I_1..I_n first, then column sets J_1..J_n."""
    shape = as_shape(shape)
    n = len(shape)
    if len(row_sizes) != n or len(col_sizes) != n:
        raise ValueError(f"need {n} row and column sizes for shape {shape}")
    total = int(np.prod(shape, dtype=np.int64))
    for m, (d, rs, cs) in enumerate(zip(shape, row_sizes, col_sizes), start=1):
        if not 1 <= int(rs) <= d:
            raise ValueError(f"mode {m}: row sample size {rs} outside [1, {d}]")
        if not 1 <= int(cs) <= total // d:
            raise ValueError(f"mode {m}: column sample size {cs} outside [1, {total // d}]")
    rows = tuple(_draw_without_replacement(rng, d, int(s)) for d, s in zip(shape, row_sizes))
    cols = tuple(_draw_without_replacement(rng, total // d, int(s)) for d, s in zip(shape, col_sizes))
    return SampleIndices(rows=rows, cols=cols)


def sample_indices(shape, ranks, upsilon, rng) -> SampleIndices:
    """fiber_cur.py:133-145."""
    rows, cols = sample_sizes(shape, ranks, upsilon)
    return draw_sample_indices(shape, rows, cols, rng)
