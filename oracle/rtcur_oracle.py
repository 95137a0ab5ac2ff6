"""CPU oracle for the RTCUR hot path -- TEST INFRASTRUCTURE, not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker (or
as the timed CPU baseline "port").  The product path in
``paper_2108_10448_b200`` never imports it.

It restates, in numpy plus one small C kernel (``gkr_svd.c``, Golub-Kahan-
Reinsch SVD), the reference solver at /root/reference/pkg/src/rtcur
(paths below are relative to that package):

* sampling      fiber_cur.py:110-130 (sizes), 148-174 (draw order), 189-209
                (without-replacement draw: permutation vs iid stream + unique)
* gather        tensor.py:235-240 (core via np.ix_), solver.py:175-182 +
                tensor.py:243-283 (fiber base offsets, strided gather)
* threshold     solver.py:195-199 -> py_kernels.py:226-230 (strict |x| > zeta)
* build         fiber_cur.py:229-274, linalg.py:46-74 (rank-r truncation,
                pinv cutoff tau = max(m, p) * sigma_1 * 1e-12)
* evaluation    fiber_cur.py:288-294 (mode-product chain), 297-326 (einsum over
                the sampled core -- the reference's hot spot, kept on purpose so
                the CPU baseline costs what the reference costs)
* error         solver.py:209-231
* loop          solver.py:260-389 (decay-before-threshold, F caches L blocks,
                R redraws and re-evaluates, stop at err <= eps)
* full output   fiber_cur.py:277-285 + cli.py:237-243

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
(scratch build of /root/reference/pkg in this container) and writes
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against every one of those vectors (indices bit-exact, HT bit-exact, blocks
and error histories within the reference's own tolerances).
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

PINV_RTOL = 1e-12  # linalg.py:23
RANK_DEFICIENCY_RTOL = 1e-8  # solver.py:64


def build_oracle_lib(force: bool = False) -> str:
    """Compile gkr_svd.c into oracle/_build/liboracle.so (gcc, -O2)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    src = os.path.join(_HERE, "gkr_svd.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess

        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", tmp, src, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        path = build_oracle_lib()
        lib = ctypes.CDLL(path)
        lib.oracle_dense_svd.restype = ctypes.c_int
        lib.oracle_dense_svd.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


# ----------------------------------------------------------------- kernels


def dense_svd(a: np.ndarray):
    """Economy SVD a == u @ diag(s) @ vt (py_kernels.py:29-54 contract)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.size == 0:
        raise ValueError(f"dense_svd expects a nonempty 2-d array, got shape {a.shape}")
    m, p = a.shape
    q = min(m, p)
    af = np.asfortranarray(a)
    u = np.zeros((m, q), order="F")
    s = np.zeros(q)
    vt = np.zeros((q, p), order="F")
    st = _load().oracle_dense_svd(af.ctypes.data, m, p, u.ctypes.data, s.ctypes.data, vt.ctypes.data)
    if st == 1:
        raise ArithmeticError("SVD failed to converge; input is likely not finite")
    if st != 0:
        raise ValueError("dense_svd: bad shape")
    return u, s, vt


def hard_threshold(a: np.ndarray, zeta: float) -> np.ndarray:
    """Keep |x| strictly above zeta (solver.py:195-199, py_kernels.py:226-230)."""
    if not zeta >= 0.0:
        raise ValueError(f"threshold must be nonnegative, got {zeta}")
    out = np.array(a, dtype=np.float64, copy=True)
    out[np.abs(out) <= zeta] = 0.0
    return out


@dataclass(frozen=True)
class TruncSvd:
    """linalg.py:26-56."""

    u: np.ndarray
    singular_values: np.ndarray
    v: np.ndarray

    def reconstruct(self) -> np.ndarray:
        return (self.u * self.singular_values) @ self.v.T

    def pinv(self) -> np.ndarray:
        s = self.singular_values
        tau = max(self.u.shape[0], self.v.shape[0]) * float(s[0]) * PINV_RTOL
        inv = np.divide(1.0, s, out=np.zeros_like(s), where=s > tau)
        return (self.v * inv) @ self.u.T


def truncated_svd(m: np.ndarray, r: int, spectrum: list | None = None) -> TruncSvd:
    """linalg.py:59-74.  ``spectrum`` (optional list) receives the full singular
    values (parity tooling logs the sigma_r / sigma_{r+1} gap from them)."""
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or m.size == 0:
        raise ValueError(f"truncated_svd needs a nonempty matrix, got shape {m.shape}")
    if not np.isfinite(m).all():
        raise ValueError("truncated_svd input contains non-finite entries")
    q = min(m.shape)
    if not 1 <= r <= q:
        raise ValueError(f"rank {r} outside [1, {q}] for shape {m.shape}")
    u, s, vt = dense_svd(m)
    if spectrum is not None:
        spectrum.append(s.copy())
    return TruncSvd(u=u[:, :r].copy(), singular_values=s[:r].copy(), v=vt[:r].T.copy())


# ----------------------------------------------------------------- layout


def strides_of(shape):
    out, acc = [], 1
    for d in shape:
        out.append(acc)
        acc *= d
    return tuple(out)


def decode_fiber_columns(shape, k, cols):
    """tensor.py:250-270 (1-based columns -> 1-based multi-index over modes != k)."""
    cols = np.asarray(cols, dtype=np.int64).reshape(-1)
    others = [d for j, d in enumerate(shape, start=1) if j != k]
    total = int(np.prod(others, dtype=np.int64)) if others else 1
    if cols.size and (cols.min() < 1 or cols.max() > total):
        raise IndexError(f"column index outside [1, {total}] for mode {k} of {shape}")
    rem = cols - 1
    out = []
    for d in others:
        out.append((rem % d) + 1)
        rem = rem // d
    return tuple(out)


def fiber_base_offsets(shape, k, cols):
    """tensor.py:273-283."""
    parts = decode_fiber_columns(shape, k, cols)
    st = strides_of(shape)
    other = [s for j, s in enumerate(st, start=1) if j != k]
    base = np.zeros(np.asarray(cols).size, dtype=np.int64)
    for idx, s in zip(parts, other):
        base += (idx - 1) * s
    return base


def gather_fibers(flat: np.ndarray, shape, k: int, cols: np.ndarray) -> np.ndarray:
    """solver.py:175-182 -> d_k x |J_k| block of mode-k fibers."""
    bases = fiber_base_offsets(shape, k, cols)
    stride = strides_of(shape)[k - 1]
    idx = bases[np.newaxis, :] + stride * np.arange(shape[k - 1], dtype=np.int64)[:, np.newaxis]
    return flat[idx]


def core_block(arr_f: np.ndarray, rows) -> np.ndarray:
    """tensor.py:235-240 (arr_f is the F-ordered n-d view)."""
    return np.asfortranarray(arr_f[np.ix_(*[r - 1 for r in rows])])


def mode_product(t: np.ndarray, a: np.ndarray, k: int) -> np.ndarray:
    """tensor.py:218-232 on plain F-ordered numpy arrays (k is 1-based)."""
    shape = t.shape
    unf = np.reshape(np.moveaxis(t, k - 1, 0), (shape[k - 1], -1), order="F")
    prod = a @ unf
    rest = tuple(d for j, d in enumerate(shape, start=1) if j != k)
    out = np.moveaxis(prod.reshape((a.shape[0],) + rest, order="F"), 0, k - 1)
    return np.asfortranarray(out)


# ----------------------------------------------------------------- sampling


def sample_sizes(shape, ranks, upsilon):
    """fiber_cur.py:110-130."""
    shape = tuple(int(d) for d in shape)
    total = int(np.prod(shape, dtype=np.int64))
    rows, cols = [], []
    for d, r in zip(shape, ranks):
        rest = total // d
        rows.append(min(d, max(r, math.ceil(upsilon * r * math.log(d)))))
        cols.append(min(rest, max(r, math.ceil(upsilon * r * math.log(rest)))))
    return tuple(rows), tuple(cols)


def draw_without_replacement(rng: np.random.Generator, population: int, k: int) -> np.ndarray:
    """fiber_cur.py:189-209 (same RNG consumption, hence identical sets)."""
    if k >= population:
        return np.arange(1, population + 1, dtype=np.int64)
    if 3 * k >= population:
        picked = rng.permutation(population)[:k]
        return np.sort(picked.astype(np.int64)) + 1
    out = np.empty(0, dtype=np.int64)
    while out.size < k:
        need = k - out.size
        batch = rng.integers(0, population, size=need + need // 2 + 16, dtype=np.int64)
        merged = np.concatenate([out, batch])
        _, first = np.unique(merged, return_index=True)
        out = merged[np.sort(first)]
    return np.sort(out[:k]) + 1


@dataclass(frozen=True)
class Sample:
    rows: tuple
    cols: tuple


def draw_sample_indices(shape, row_sizes, col_sizes, rng) -> Sample:
    """fiber_cur.py:148-174: all row sets first, then all column sets."""
    shape = tuple(int(d) for d in shape)
    total = int(np.prod(shape, dtype=np.int64))
    for m, (d, rs, cs) in enumerate(zip(shape, row_sizes, col_sizes), start=1):
        if not 1 <= int(rs) <= d:
            raise ValueError(f"mode {m}: row sample size {rs} outside [1, {d}]")
        if not 1 <= int(cs) <= total // d:
            raise ValueError(f"mode {m}: column sample size {cs} outside [1, {total // d}]")
    rows = tuple(draw_without_replacement(rng, d, int(s)) for d, s in zip(shape, row_sizes))
    cols = tuple(draw_without_replacement(rng, total // d, int(s)) for d, s in zip(shape, col_sizes))
    return Sample(rows=rows, cols=cols)


# ----------------------------------------------------------------- CUR


@dataclass(frozen=True)
class OracleCur:
    core: np.ndarray
    fibers: tuple
    intersections: tuple
    indices: Sample
    factors: tuple
    spectra: tuple = ()   # full singular values of each intersection (diagnostics only)


def assemble(core: np.ndarray, fibers, idx: Sample, ranks) -> OracleCur:
    """fiber_cur.py:229-274."""
    inters, factors, spectra = [], [], []
    for rows, rk, fib in zip(idx.rows, ranks, fibers):
        if rk > rows.size or rk > fib.shape[1]:
            raise ValueError(f"rank {rk} exceeds sample sizes")
        inter = truncated_svd(fib[rows - 1, :], rk, spectra)
        inters.append(inter)
        factors.append(fib @ inter.pinv())
    return OracleCur(core=core, fibers=tuple(fibers), intersections=tuple(inters),
                     indices=idx, factors=tuple(factors), spectra=tuple(spectra))


def eval_subtensor(cur: OracleCur, rows) -> np.ndarray:
    """fiber_cur.py:288-294."""
    out = cur.core
    for m, (fac, r) in enumerate(zip(cur.factors, rows), start=1):
        out = mode_product(out, fac[r - 1, :], m)
    return out


def eval_fibers_einsum(cur: OracleCur, k: int, cols) -> np.ndarray:
    """fiber_cur.py:297-326 verbatim in structure: one ``np.einsum`` over the
    |I_1|x...x|I_n| core and the other modes' factor rows, then ``factor_k @``.
    This is the reference's hot spot; the CPU baseline ("port") times it."""
    shape = tuple(f.shape[0] for f in cur.fibers)
    n = len(shape)
    cols = np.asarray(cols, dtype=np.int64).reshape(-1)
    parts = decode_fiber_columns(shape, k, cols)
    core = cur.core
    other = [m for m in range(1, n + 1) if m != k]
    if not other:
        small = np.repeat(core.reshape(-1, 1), cols.size, axis=1)
        return cur.factors[k - 1] @ small
    ops = [core, list(range(n))]
    for m, r in zip(other, parts):
        ops.append(cur.factors[m - 1][r - 1, :])
        ops.append([n, m - 1])
    small = np.einsum(*ops, [k - 1, n], optimize=True)
    return cur.factors[k - 1] @ small


def eval_fibers_blas(cur: OracleCur, k: int, cols, chunk_bytes: int = 1 << 28) -> np.ndarray:
    """The same contraction as ``eval_fibers_einsum`` (fiber_cur.py:318-326:
    small[:, j] = sum over the other modes' core indices of core * prod_m
    factor_m[i_m(j), :]), associated explicitly: one BLAS GEMM against the
    first other mode's factor rows, then one batched dot per remaining mode,
    columns in chunks of ``chunk_bytes`` of intermediate.  Same sum, different
    association: agrees with the einsum to ~1e-15 relative
    (tests/test_oracle_golden.py::test_eval_fibers_blas_matches_einsum) and is
    15-40x faster, which is what makes full-size oracle solves at BASELINE
    configs 1-4 feasible for the parity runs."""
    shape = tuple(f.shape[0] for f in cur.fibers)
    n = len(shape)
    cols = np.asarray(cols, dtype=np.int64).reshape(-1)
    parts = decode_fiber_columns(shape, k, cols)
    core = cur.core
    other = [m for m in range(1, n + 1) if m != k]
    if not other:
        small = np.repeat(core.reshape(-1, 1), cols.size, axis=1)
        return cur.factors[k - 1] @ small
    J = cols.size
    small = np.empty((core.shape[k - 1], J))
    m1 = other[0]
    per_col = 8 * (core.size // core.shape[m1 - 1])
    step = max(1, min(J, chunk_bytes // max(per_col, 1))) if J else 1
    for j0 in range(0, J, step):
        j1 = min(J, j0 + step)
        rows1 = cur.factors[m1 - 1][parts[0][j0:j1] - 1, :]          # (jc, |I_m1|)
        t = np.tensordot(rows1, core, axes=([1], [m1 - 1]))          # (jc, modes != m1 ascending)
        axes = [m for m in range(1, n + 1) if m != m1]               # t axis i+1 <-> mode axes[i]
        for m, r in zip(other[1:], parts[1:]):
            rows = cur.factors[m - 1][r[j0:j1] - 1, :]                # (jc, |I_m|)
            t = np.moveaxis(t, axes.index(m) + 1, -1)
            lead = t.shape[:-1]
            t = np.matmul(t.reshape(lead[0], -1, t.shape[-1]), rows[:, :, None]).reshape(lead)
            axes.remove(m)
        small[:, j0:j1] = t.T
    return cur.factors[k - 1] @ small


# which evaluation the oracle's solve uses: "blas" (parity runs, default) or
# "einsum" (the CPU baseline that costs what the reference costs)
EVAL_MODE = os.environ.get("RTCUR_ORACLE_EVAL", "blas")


def eval_fibers(cur: OracleCur, k: int, cols, mode: str | None = None) -> np.ndarray:
    """fiber_cur.py:297-326."""
    if (mode or EVAL_MODE) == "einsum":
        return eval_fibers_einsum(cur, k, cols)
    return eval_fibers_blas(cur, k, cols)


def eval_blocks(cur: OracleCur, idx: Sample, mode: str | None = None):
    """solver.py:242-249."""
    core = eval_subtensor(cur, idx.rows)
    fibers = [eval_fibers(cur, k, c, mode) for k, c in enumerate(idx.cols, start=1)]
    return core, fibers


def reconstruct_full(cur: OracleCur) -> np.ndarray:
    """fiber_cur.py:277-285 (F-ordered n-d array)."""
    out = cur.core
    for m, fac in enumerate(cur.factors, start=1):
        out = mode_product(out, fac, m)
    return out


def _block_norm(core, fibers) -> float:
    total = float(np.sqrt(np.sum(core * core)))
    for f in fibers:
        total += float(np.sqrt(np.sum(f * f)))
    return total


def sampled_relative_error(e_core, e_fibers, x_core, x_fibers) -> float:
    """solver.py:216-231."""
    num = _block_norm(e_core, e_fibers)
    den = _block_norm(x_core, x_fibers)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / den


def deficiency_flags(cur: OracleCur):
    """solver.py:252-257."""
    out = []
    for inter in cur.intersections:
        s = inter.singular_values
        out.append(bool(s[0] <= 0.0 or s[-1] <= RANK_DEFICIENCY_RTOL * s[0]))
    return tuple(out)


# ----------------------------------------------------------------- solver


@dataclass
class OracleResult:
    cur: OracleCur
    s_core: np.ndarray
    s_fibers: tuple
    indices: Sample
    error_history: tuple
    iterations: int
    converged: bool
    diagnostics: tuple
    zeta_final: float
    timings: dict
    trace: list = field(default_factory=list)
    iter_times: list = field(default_factory=list)


def inf_norm(flat: np.ndarray) -> float:
    """solver.py:184-192 (chunked max |x|)."""
    best = 0.0
    step = 1 << 18
    for start in range(0, flat.size, step):
        best = max(best, float(np.max(np.abs(flat[start:start + step]))))
    return best


def iter_solve(x_flat: np.ndarray, shape, ranks, *, eps=1e-5, zeta0=None, gamma=0.7, upsilon=3.0,
               variant="F", max_iters=500, seed=None, row_sample_sizes=None, col_sample_sizes=None,
               iteration_budget_s: float | None = None, eval_mode: str | None = None, stats: dict | None = None):
    """solver.py:260-389 restated as a generator: yields one dict per iteration
    (iteration, zeta, indices, x/s/l blocks, error, flags, cur).  ``stats``
    (optional dict) receives timings / iter_times / converged as they happen.
    x_flat is the mode-1-fastest float64 buffer.

    iteration_budget_s (CPU-baseline use only) stops after the first iteration
    that pushes the elapsed loop time past the budget."""
    shape = tuple(int(d) for d in shape)
    x_flat = np.ascontiguousarray(x_flat, dtype=np.float64).reshape(-1)
    arr = x_flat.reshape(shape, order="F")
    variant = variant.upper()
    st = stats if stats is not None else {}
    timings = st.setdefault("timings", {k: 0.0 for k in ("sample", "gather", "eval_lowrank", "threshold",
                                                           "build", "error", "total")})
    iter_times = st.setdefault("iter_times", [])
    st["converged"] = False
    t_start = time.perf_counter()
    rng = np.random.default_rng(seed)
    rows, cols = sample_sizes(shape, ranks, upsilon)
    if row_sample_sizes is not None:
        rows = tuple(row_sample_sizes)
    if col_sample_sizes is not None:
        cols = tuple(col_sample_sizes)

    def gather(idx):
        core = core_block(arr, idx.rows)
        fibers = [gather_fibers(x_flat, shape, k, c) for k, c in enumerate(idx.cols, start=1)]
        return core, fibers

    t0 = time.perf_counter()
    idx = draw_sample_indices(shape, rows, cols, rng)
    timings["sample"] += time.perf_counter() - t0
    t0 = time.perf_counter()
    x_core, x_fibers = gather(idx)
    timings["gather"] += time.perf_counter() - t0
    zeta = float(zeta0) if zeta0 is not None else inf_norm(x_flat)
    t_loop = time.perf_counter()

    lcur = None
    lblocks = None
    for k in range(1, max_iters + 1):
        t_iter = time.perf_counter()
        if variant == "R" and k >= 2:
            t0 = time.perf_counter()
            idx = draw_sample_indices(shape, rows, cols, rng)
            timings["sample"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            x_core, x_fibers = gather(idx)
            timings["gather"] += time.perf_counter() - t0
            lblocks = None
        zeta *= gamma
        t0 = time.perf_counter()
        if lcur is None:
            l_core = np.zeros_like(x_core)
            l_fibers = [np.zeros_like(f) for f in x_fibers]
        elif lblocks is None:
            l_core, l_fibers = eval_blocks(lcur, idx, eval_mode)
        else:
            l_core, l_fibers = lblocks
        prev_l = (l_core, l_fibers)
        timings["eval_lowrank"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        s_core = hard_threshold(x_core - l_core, zeta)
        s_fibers = [hard_threshold(xf - lf, zeta) for xf, lf in zip(x_fibers, l_fibers)]
        timings["threshold"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        clean_core = np.asfortranarray(x_core - s_core)
        clean_fibers = tuple(xf - sf for xf, sf in zip(x_fibers, s_fibers))
        lcur = assemble(clean_core, clean_fibers, idx, ranks)
        fl = deficiency_flags(lcur)
        timings["build"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        l_core, l_fibers = eval_blocks(lcur, idx, eval_mode)
        lblocks = (l_core, l_fibers)
        e_core = x_core - l_core - s_core
        e_fibers = [xf - lf - sf for xf, lf, sf in zip(x_fibers, l_fibers, s_fibers)]
        err = sampled_relative_error(e_core, e_fibers, x_core, x_fibers)
        timings["error"] += time.perf_counter() - t0
        iter_times.append(time.perf_counter() - t_iter)
        done = err <= eps
        st["converged"] = bool(done)
        timings["total"] = time.perf_counter() - t_start
        timings["loop"] = time.perf_counter() - t_loop
        yield {"iteration": k, "zeta": zeta, "indices": idx, "x_core": x_core, "x_fibers": tuple(x_fibers),
               "s_core": s_core, "s_fibers": tuple(s_fibers), "l_core": l_core, "l_fibers": tuple(l_fibers),
               "l_prev": prev_l, "error": err, "flags": fl, "cur": lcur}
        if done:
            break
        if iteration_budget_s is not None and time.perf_counter() - t_loop > iteration_budget_s:
            break


def solve(x_flat: np.ndarray, shape, ranks, *, eps=1e-5, zeta0=None, gamma=0.7, upsilon=3.0,
          variant="F", max_iters=500, seed=None, row_sample_sizes=None, col_sample_sizes=None,
          record_trace=False, iteration_budget_s: float | None = None,
          eval_mode: str | None = None) -> OracleResult:
    """solver.py:260-389 restated (collects ``iter_solve``)."""
    stats: dict = {}
    history, flags, trace = [], [], []
    last = None
    for it in iter_solve(x_flat, shape, ranks, eps=eps, zeta0=zeta0, gamma=gamma, upsilon=upsilon,
                         variant=variant, max_iters=max_iters, seed=seed, row_sample_sizes=row_sample_sizes,
                         col_sample_sizes=col_sample_sizes, iteration_budget_s=iteration_budget_s,
                         eval_mode=eval_mode, stats=stats):
        history.append(it["error"])
        flags.append(it["flags"])
        if record_trace:
            trace.append({k: it[k] for k in ("iteration", "zeta", "indices", "s_core", "s_fibers", "l_core",
                                             "l_fibers", "error")})
        last = it
    return OracleResult(cur=last["cur"], s_core=last["s_core"], s_fibers=last["s_fibers"],
                        indices=last["indices"], error_history=tuple(history), iterations=len(history),
                        converged=stats["converged"], diagnostics=tuple(flags), zeta_final=last["zeta"],
                        timings=stats["timings"], trace=trace, iter_times=stats["iter_times"])


def full_output(x_flat: np.ndarray, shape, cur: OracleCur, zeta_final: float):
    """cli.py:237-243: L = cur_reconstruct_full(cur); S = HT(x - L, zeta_final).

    Returns flat (mode-1-fastest) L and S plus the residual sums the GPU K3
    kernel reports: sum((x - L - S)^2) and sum(x^2).
    """
    low = reconstruct_full(cur).reshape(-1, order="F")
    sp = hard_threshold(x_flat - low, zeta_final)
    resid = x_flat - low - sp
    return low, sp, float(np.sum(resid * resid)), float(np.sum(x_flat * x_flat))
