"""Batched sweeps on one GPU (reference synth.py:138-336).

``run_phase_transition`` and ``run_timing`` keep the reference's signatures,
seeds (``_trial_seeds``: SeedSequence([base_seed, *path])), instance law
(``make_instance`` on the device) and success / censoring rules.  The
difference is scheduling: independent trials are many small solves, so they
run concurrently -- ``workers`` host threads, each with its own CUDA stream and
its own pooled engines (ctypes releases the GIL in every native call and
while an iteration is awaited), filling the GPU that one small solve cannot.
Results are assembled in the reference's deterministic order, so the output
does not depend on the completion order.
"""

from __future__ import annotations

import ctypes
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .synth import InstanceSpec, make_instance_device

__all__ = ["DEFAULT_ALPHAS", "DEFAULT_UPSILONS", "METHOD_NAMES", "PhaseGrid", "TimingRow", "timing_to_csv",
           "run_phase_transition", "run_timing"]

DEFAULT_ALPHAS = tuple(round(0.05 * i, 2) for i in range(1, 13))  # synth.py:37
DEFAULT_UPSILONS = (1.0, 2.0, 3.0, 4.0, 5.0, 6.0)                  # synth.py:38
METHOD_NAMES = ("rtcur-f", "rtcur-r", "hosvd-ap")                  # synth.py:39


@dataclass(frozen=True)
class PhaseGrid:
    """Success counts over an (outlier fraction) x (oversampling) grid (synth.py:138-155)."""

    alphas: tuple
    upsilons: tuple
    trials: int
    successes: tuple  # [alpha index][upsilon index]

    def success_rate(self, i: int, j: int) -> float:
        return self.successes[i][j] / self.trials

    def to_csv(self) -> str:
        lines = ["alpha,upsilon,successes,trials"]
        for a, row in zip(self.alphas, self.successes):
            for u, s in zip(self.upsilons, row):
                lines.append(f"{a:g},{u:g},{s},{self.trials}")
        return "\n".join(lines) + "\n"


@dataclass(frozen=True)
class TimingRow:
    """One benchmark cell (synth.py:218-227)."""

    d: int
    method: str
    mean_s: float
    std_s: float
    iters: float
    censored: bool


def timing_to_csv(rows) -> str:   # synth.py:230-237
    lines = ["d,method,mean_s,std_s,iters,censored"]
    for row in rows:
        lines.append(f"{row.d},{row.method},{row.mean_s},{row.std_s},{row.iters},{int(row.censored)}")
    return "\n".join(lines) + "\n"


def _trial_seeds(base_seed: int, *path: int):   # synth.py:151-154
    state = np.random.SeedSequence([int(base_seed), *[int(p) for p in path]])
    a, b = state.generate_state(2)
    return int(a), int(b)


def _inf_norm_dev(t) -> float:
    import torch

    lib = nat.load()
    scratch = torch.empty(2, dtype=torch.float64, device=t.flat.device)
    out = ctypes.c_double()
    nat.check(lib.rtcur_abs_max(t.flat.data_ptr(), 0 if t.flat.dtype == torch.float64 else 1, t.flat.numel(),
                                scratch.data_ptr(), ctypes.byref(out), torch.cuda.current_stream().cuda_stream))
    return out.value


class _StreamPool:
    """One CUDA stream per worker thread (created lazily)."""

    def __init__(self):
        import threading

        self._local = threading.local()

    def stream(self):
        import torch

        s = getattr(self._local, "s", None)
        if s is None:
            s = self._local.s = torch.cuda.Stream()
        return s


def _run_parallel(jobs, workers):
    """jobs: list of callables -> list of results in order, run on `workers` streams."""
    import torch

    streams = _StreamPool()

    def wrap(fn):
        def run():
            s = streams.stream()
            with torch.cuda.stream(s):
                out = fn()
                s.synchronize()
            return out
        return run

    if workers <= 1:
        return [wrap(f)() for f in jobs]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        futs = [ex.submit(wrap(f)) for f in jobs]
        return [f.result() for f in futs]


def run_phase_transition(alphas=DEFAULT_ALPHAS, upsilons=DEFAULT_UPSILONS, trials: int = 10, n: int = 3, d: int = 60,
                         r: int = 3, variant: str = "F", eps: float = 1e-5, gamma: float = 0.7, max_iters: int = 150,
                         success_tol: float = 1e-3, base_seed: int = 0, progress=None, workers: int = 4) -> PhaseGrid:
    """synth.py:159-215: success when the reconstructed low-rank part is within
    success_tol relative Frobenius error of the truth; a trial that raises or
    does not converge... counts as the reference counts it (exceptions are
    failures, never aborts)."""
    import torch

    from .full import full_output
    from .solver import SolverConfig, rtcur

    alphas = tuple(float(a) for a in alphas)
    upsilons = tuple(float(u) for u in upsilons)
    if trials < 1:
        raise ValueError(f"trials must be >= 1, got {trials}")

    def trial(ia, iu, t):
        def run():
            alpha, upsilon = alphas[ia], upsilons[iu]
            inst_seed, solver_seed = _trial_seeds(base_seed, ia, iu, t)
            spec = InstanceSpec(n=n, d=d, r=r, alpha=alpha, seed=inst_seed)
            x, low, _ = make_instance_device(spec)
            ok = False
            try:
                cfg = SolverConfig(ranks=spec.ranks, eps=eps, zeta0=_inf_norm_dev(low), gamma=gamma, upsilon=upsilon,
                                   variant=variant, max_iters=max_iters, seed=solver_seed)
                res = rtcur(x, cfg)
                est, _, _ = full_output(res, want_S=False)
                diff = torch.linalg.vector_norm(low.flat - est.flat.double())
                rel = float(diff / torch.linalg.vector_norm(low.flat))
                ok = bool(rel <= success_tol)
            except Exception:
                ok = False
            return ok
        return run

    cells = [(ia, iu, t) for ia in range(len(alphas)) for iu in range(len(upsilons)) for t in range(trials)]
    results = _run_parallel([trial(*c) for c in cells], workers)
    wins = {}
    for (ia, iu, t), ok in zip(cells, results):
        wins[(ia, iu)] = wins.get((ia, iu), 0) + int(ok)
        if progress is not None:
            progress(alphas[ia], upsilons[iu], t, ok)
    grid = tuple(tuple(wins[(ia, iu)] for iu in range(len(upsilons))) for ia in range(len(alphas)))
    return PhaseGrid(alphas=alphas, upsilons=upsilons, trials=trials, successes=grid)


def _solve_timed(method, x, low, spec, solver_seed, *, eps, gamma, upsilon, max_iters):   # synth.py:240-262
    import torch

    from .hosvd_ap import ap_hosvd_trpca
    from .solver import SolverConfig, rtcur

    zeta0 = _inf_norm_dev(low)
    torch.cuda.current_stream().synchronize()
    t0 = time.perf_counter()
    if method in ("rtcur-f", "rtcur-r"):
        cfg = SolverConfig(ranks=spec.ranks, eps=eps, zeta0=zeta0, gamma=gamma, upsilon=upsilon,
                           variant="F" if method == "rtcur-f" else "R", max_iters=max_iters, seed=solver_seed)
        iters = rtcur(x, cfg).iterations
    elif method == "hosvd-ap":
        _, _, history = ap_hosvd_trpca(x, spec.ranks, zeta0=zeta0, gamma=gamma, eps=eps, max_iters=max_iters)
        iters = len(history)
    else:
        raise ValueError(f"unknown method {method!r}, expected one of {METHOD_NAMES}")
    torch.cuda.current_stream().synchronize()
    return time.perf_counter() - t0, iters


def run_timing(dims, methods=METHOD_NAMES, repeats: int = 3, n: int = 3, r: int = 3, alpha: float = 0.1,
               upsilon: float = 3.0, eps: float = 1e-5, gamma: float = 0.7, max_iters: int = 500,
               timeout_s: float | None = None, base_seed: int = 0, progress=None):
    """synth.py:265-336: wall-clock per method and size on identical instances.
    Timed solves run one at a time (a timing sweep measures each solve alone)."""
    dims = tuple(int(d) for d in dims)
    methods = tuple(methods)
    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    for m in methods:
        if m not in METHOD_NAMES:
            raise ValueError(f"unknown method {m!r}, expected one of {METHOD_NAMES}")
    rows = []
    for di, d in enumerate(dims):
        for method in methods:
            times, iter_counts = [], []
            censored = False
            spent = 0.0
            for rep in range(repeats):
                inst_seed, solver_seed = _trial_seeds(base_seed, di, rep)
                spec = InstanceSpec(n=n, d=d, r=r, alpha=alpha, seed=inst_seed)
                x, low, _ = make_instance_device(spec)
                elapsed, iters = _solve_timed(method, x, low, spec, solver_seed, eps=eps, gamma=gamma, upsilon=upsilon,
                                              max_iters=max_iters)
                times.append(elapsed)
                iter_counts.append(iters)
                spent += elapsed
                if progress is not None:
                    progress(d, method, rep, elapsed)
                if timeout_s is not None and spent > timeout_s:
                    censored = rep + 1 < repeats
                    break
            rows.append(TimingRow(d=d, method=method, mean_s=float(np.mean(times)), std_s=float(np.std(times)),
                                  iters=float(np.mean(iter_counts)), censored=censored))
    return rows
