"""Step 5 of the north star: the full-tensor reconstruction L and outlier
tensor S, i.e. the reference's ``rtcur solve --full-output`` step
(/root/reference/pkg/src/rtcur/cli.py:237-243):

    L = cur_reconstruct_full(res.cur)              (fiber_cur.py:277-285)
    S = hard_threshold(x - L, res.zeta_final)

run by the streaming K3 kernel (k_full.cu) from the collapsed Tucker form,
with the residual sums sum((x-L-S)^2) and sum(x^2) fused in.
"""

from __future__ import annotations

import numpy as np

from .tensor import DenseTensor, DeviceTensor

__all__ = ["full_output", "cur_reconstruct_full"]


def _engine_of(res_or_cur):
    cur = getattr(res_or_cur, "cur", res_or_cur)
    eng = getattr(cur, "_engine", None)
    if eng is None:
        raise ValueError("this FiberCur was not produced by paper_2108_10448_b200.rtcur (no device state)")
    return eng


def full_output(res, x=None, want_L: bool = True, want_S: bool = True):
    """Full L and S (DeviceTensors, dtype of X) plus the full relative residual
    ||X - L - S||_F / ||X||_F.  ``x`` defaults to the tensor the solve ran on."""
    eng = _engine_of(res)
    if x is not None:
        dev = x if isinstance(x, DeviceTensor) else DeviceTensor.from_host(x)
        eng.bind(dev.flat)
    L, S, e2, x2 = eng.full_output(res.zeta_final, want_L=want_L, want_S=want_S)
    lo, hi = eng.slab   # a sharded engine reconstructs its mode-1 slab (residual of the slab only;
    shape = (hi - lo,) + tuple(eng.shape[1:])   # dist.full_output_sharded all-reduces the global one)
    rel = float(np.sqrt(e2) / np.sqrt(x2)) if x2 > 0 else (0.0 if e2 == 0 else float("inf"))
    return (DeviceTensor(L, shape) if L is not None else None,
            DeviceTensor(S, shape) if S is not None else None, rel)


def cur_reconstruct_full(cur) -> DenseTensor:
    """fiber_cur.py:277-285: materialise core x_i factors[i] (host DenseTensor)."""
    eng = _engine_of(cur)
    saved = eng._x
    eng.unbind()
    try:
        L, _, _, _ = eng.full_output(0.0, want_L=True, want_S=False)
    finally:
        if saved is not None:
            eng.bind(saved)
    return DeviceTensor(L, eng.shape).to_dense()
