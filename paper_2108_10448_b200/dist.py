"""Mode-1 slab sharding over NCCL.

Rank p holds X[lo_p:hi_p, ...] (``synth.slab_bounds``: contiguous, sizes
differ by at most one row).  Per solve:

* zeta_0      local K0 abs-max, ``all_reduce(MAX)`` of one scalar;
* gather      K1 gather writes the entries whose mode-1 index the rank owns
              (zeros elsewhere); ``all_reduce(SUM)`` of the compact blocks
              reproduces the full gather bit-exactly -- once for RTCUR-F,
              every iteration for RTCUR-R (the reference's per-iteration
              regather, solver.py:315-322);
* the small CUR build, the error sums and the stop rule then run replicated
  and identically on every rank (deterministic kernels, same inputs);
* full output K3 runs on the local slab; the two residual sums are
  ``all_reduce(SUM)``-ed.

One process per GPU (torchrun), backend "nccl".
"""

from __future__ import annotations

import numpy as np

from .solver import SolverConfig, SolveResult, _solve, _Source
from .synth import slab_bounds
from .tensor import DeviceTensor

__all__ = ["rtcur_sharded", "full_output_sharded", "slab_bounds"]


def rtcur_sharded(x_slab: DeviceTensor, global_shape, slab, cfg: SolverConfig, record_trace: bool = False,
                  group=None) -> SolveResult:
    """rtcur() on a mode-1-sharded tensor: ``x_slab`` is this rank's slab
    [lo, hi) of a ``global_shape`` tensor."""
    return _solve(_Source(x_slab, slab=tuple(slab), group=group, global_shape=tuple(global_shape)), cfg,
                  record_trace)


def full_output_sharded(res: SolveResult, group=None):
    """K3 on the local slab: (L_slab, S_slab, global ||X - L - S|| / ||X||)."""
    import torch
    import torch.distributed as dist

    eng = res.cur._engine
    L, S, e2, x2 = eng.full_output(res.zeta_final)
    t = torch.tensor([e2, x2], dtype=torch.float64, device=eng.device)
    if group is not None or (dist.is_available() and dist.is_initialized()):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    e2, x2 = float(t[0]), float(t[1])
    rel = float(np.sqrt(e2) / np.sqrt(x2)) if x2 > 0 else (0.0 if e2 == 0 else float("inf"))
    lo, hi = eng.slab
    shape = (hi - lo,) + tuple(eng.shape[1:])
    return DeviceTensor(L, shape), (DeviceTensor(S, shape) if S is not None else None), rel
