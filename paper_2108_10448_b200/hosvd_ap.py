"""Dense HOSVD alternating projections on the GPU -- the paper's comparison
baseline (reference /root/reference/pkg/src/rtcur/reference.py:132-193).

Same loop as the reference: zeta <- gamma zeta, S = HT(X - L, zeta),
L = HOSVD_r(X - S) reconstructed, stop when ||X - L - S||_F / ||X||_F <= eps.
Every step touches the whole tensor in HBM:

* threshold + C = X - S and the residual sums: native fused passes
  (``rtcur_ap_threshold``, ``rtcur_ap_residual``, fixed-order reductions);
* the mode-m Grams C_(m) C_(m)^T and the mode products: plain fp64 GEMMs
  (cuBLAS through torch.tensordot -- library GEMMs, allowed for the baseline);
* the top-r_m eigenvectors of each Gram: ``torch.linalg.eigh`` (cuSOLVER).

The HOSVD reconstruction core x_m U_m with core = C x_m U_m^T equals
C x_m (U_m U_m^T): it depends only on the leading subspaces, so the Gram
eigenvectors give the same L as the reference's SVD of each unfolding.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .tensor import DenseTensor, DeviceTensor

__all__ = ["hosvd_device", "ap_hosvd_trpca"]


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _tview(flat, shape):
    # C-order view with reversed axes of an F-order (mode-1 fastest) buffer: axis n-1-m is mode m
    return flat.reshape(tuple(reversed(shape)))


def _mode_product(t, mat, m, n):
    """t x_m mat (mat: new_d x d_m) on the reversed-axes view."""
    import torch

    ax = n - 1 - m
    out = torch.tensordot(mat, t, dims=([1], [ax]))   # new axis first
    return torch.movedim(out, 0, ax)


def hosvd_device(c_flat, shape, ranks):
    """Leading r_m left singular vectors of every unfolding of C (F-order flat
    fp64 CUDA tensor), from the mode Grams.  Returns [U_m (d_m x r_m)]."""
    import torch

    n = len(shape)
    t = _tview(c_flat, shape)
    factors = []
    for m in range(n):
        ax = n - 1 - m
        others = [a for a in range(n) if a != ax]
        G = torch.tensordot(t, t, dims=(others, others)) if others else torch.outer(t, t)
        w, v = torch.linalg.eigh(G)
        factors.append(v[:, -ranks[m]:].flip(1).contiguous())   # descending
    return factors


def _reconstruct(c_flat, shape, factors):
    import torch

    n = len(shape)
    t = _tview(c_flat, shape)
    for m, U in enumerate(factors):
        t = _mode_product(t, U.T.contiguous(), m, n)
    for m, U in enumerate(factors):
        t = _mode_product(t, U, m, n)
    return t.contiguous().reshape(-1)


def ap_hosvd_trpca(x, ranks, zeta0=None, gamma: float = 0.7, eps: float = 1e-5, max_iters: int = 500):
    """reference.py:145-193 on the GPU.  ``x``: DeviceTensor / DenseTensor (fp64
    math; fp32 inputs are upcast).  Returns (low, sparse, history) with low/sparse
    fp64 DeviceTensors and history the per-iteration relative residuals."""
    import torch

    if not 0.0 < gamma < 1.0:
        raise ValueError(f"gamma must lie in (0, 1), got {gamma}")
    if not eps > 0.0:
        raise ValueError(f"eps must be positive, got {eps}")
    if isinstance(x, DenseTensor):
        x = DeviceTensor.from_host(x)
    shape = tuple(int(d) for d in x.shape)
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != len(shape):
        raise ValueError(f"{len(ranks)} ranks for a {len(shape)}-mode tensor")
    for m, (r, d) in enumerate(zip(ranks, shape), start=1):
        if not 1 <= r <= d:
            raise ValueError(f"mode {m}: rank {r} outside [1, {d}]")
    lib = nat.load()
    X = x.flat if x.flat.dtype == torch.float64 else x.flat.double()
    N = X.numel()
    scratch = torch.empty(1300, dtype=torch.float64, device=X.device)
    if zeta0 is None:
        zm = ctypes.c_double()
        nat.check(lib.rtcur_abs_max(X.data_ptr(), 0, N, scratch.data_ptr(), ctypes.byref(zm), _stream()))
        zeta = zm.value
    else:
        zeta = float(zeta0)
    if zeta < 0.0:
        raise ValueError(f"zeta0 must be nonnegative, got {zeta}")
    L = torch.zeros_like(X)
    S = torch.empty_like(X)
    C = torch.empty_like(X)
    sums = (ctypes.c_double * 2)()
    history = []
    first = True
    for _ in range(int(max_iters)):
        zeta *= gamma
        nat.check(lib.rtcur_ap_threshold(X.data_ptr(), None if first else L.data_ptr(), N, zeta, S.data_ptr(),
                                         C.data_ptr(), _stream()))
        first = False
        factors = hosvd_device(C, shape, ranks)
        L = _reconstruct(C, shape, factors)
        nat.check(lib.rtcur_ap_residual(X.data_ptr(), L.data_ptr(), S.data_ptr(), N, scratch.data_ptr(), sums,
                                        _stream()))
        e2, x2 = float(sums[0]), float(sums[1])
        err = float(np.sqrt(e2))
        xn = float(np.sqrt(x2))
        err = 0.0 if xn == 0.0 and err == 0.0 else (float("inf") if xn == 0.0 else err / xn)
        history.append(err)
        if err <= eps:
            break
    return DeviceTensor(L, shape), DeviceTensor(S.clone(), shape), history
