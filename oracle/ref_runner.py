"""Run the REAL reference package (built into oracle/_ref by build_ref.sh) on a
seeded instance -- TEST / BASELINE INFRASTRUCTURE, never product code.

Only ``bench.py`` (the ``--impl reference`` arm and the ``cpu_baseline`` leg)
and ``tests/`` use this module.  It drives the reference exclusively through
its public API: ``rtcur.rtcur(accessor, SolverConfig(...))`` with the
reference's own ``DenseTensorAccessor`` (/root/reference/pkg/src/rtcur/
solver.py:160-192, 260-389) and ``RTCUR_BACKEND=compiled`` (its Cython
kernels, _backend/__init__.py:10-33), i.e. the stock code path.

Per-iteration times come from a pass-through accessor (the reference's
``TensorAccessor`` protocol, solver.py:144-159): RTCUR-R re-gathers the core
block at the start of every iteration (solver.py:315-322), so the times of
successive ``core_block`` calls delimit iterations; the solve's return closes
the last one.  RTCUR-F gathers once, so its loop time is ``timings['total']``
minus the setup the reference itself reports (sample + gather) and the
``inf_norm`` scan the accessor times (the same per-iteration meaning).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")

_mod = None


def available() -> bool:
    d = os.path.join(REF_DIR, "rtcur", "_backend")
    return os.path.isdir(d) and any(f.startswith("_core") and f.endswith(".so") for f in os.listdir(d))


def import_reference():
    """The reference package from oracle/_ref with its compiled backend."""
    global _mod
    if _mod is not None:
        return _mod
    if not available():
        raise ImportError(f"reference not built in {REF_DIR} (run oracle/build_ref.sh where /root/reference exists)")
    os.environ["RTCUR_BACKEND"] = "compiled"
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import rtcur  # noqa: E402

    if rtcur._backend.backend_name != "compiled":
        raise ImportError(f"reference backend is {rtcur._backend.backend_name!r}, expected 'compiled'")
    _mod = rtcur
    return rtcur


def _digest(a) -> str:
    return hashlib.sha256(np.packbits(np.asarray(a).reshape(-1, order="F") != 0.0).tobytes()).hexdigest()


def run(x_flat, shape, ranks, *, eps, variant, max_iters, seed, row_sample_sizes, col_sample_sizes,
        gamma=0.7, zeta0=None):
    """One reference solve; returns (SolveResult, info) where info holds the
    per-iteration wall times, the setup time and the host thread budget."""
    rtcur = import_reference()
    from rtcur import DenseTensor, SolverConfig
    from rtcur.solver import DenseTensorAccessor

    inner = DenseTensorAccessor(DenseTensor(np.asarray(x_flat, dtype=np.float64), tuple(shape)))
    marks: list = []
    scan = [0.0]

    class TimedAccessor:
        """Pass-through TensorAccessor recording when each gather starts."""

        @property
        def shape(self):
            return inner.shape

        def core_block(self, rows):
            marks.append(time.perf_counter())
            return inner.core_block(rows)

        def fiber_block(self, k, cols):
            return inner.fiber_block(k, cols)

        def inf_norm(self):
            t = time.perf_counter()
            v = inner.inf_norm()
            scan[0] += time.perf_counter() - t
            return v

    cfg = SolverConfig(ranks=tuple(ranks), eps=eps, zeta0=zeta0, gamma=gamma, variant=variant, max_iters=max_iters,
                       seed=seed, row_sample_sizes=tuple(row_sample_sizes), col_sample_sizes=tuple(col_sample_sizes))
    t0 = time.perf_counter()
    res = rtcur.rtcur(TimedAccessor(), cfg)
    t_end = time.perf_counter()
    if variant.upper() == "R":
        # iteration k >= 2 runs from its own gather to the next one (or the return);
        # iteration 1's start is hidden behind the initial gather + scan: not timed
        ends = marks[1:res.iterations] + [t_end]
        iter_times = [None] + [ends[k] - marks[k] for k in range(1, res.iterations)]
    else:
        loop = res.timings["total"] - res.timings["sample"] - res.timings["gather"] - scan[0]
        iter_times = [loop / res.iterations] * res.iterations
    info = {"iter_times": iter_times, "wall_s": t_end - t0, "inf_norm_s": scan[0],
            "setup_s": res.timings["sample"] + res.timings["gather"] + scan[0],
            "threads": int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1)),
            "error_history": [float(e) for e in res.error_history],
            "s_core_support_sha256": _digest(res.sparse.core),
            "s_fibers_support_sha256": [_digest(f) for f in res.sparse.fibers],
            "backend": rtcur._backend.backend_name}
    return res, info
