"""Mode-1 slab sharding over torch.distributed.

Rank p holds X[lo_p:hi_p, ...] (``synth.slab_bounds``: contiguous, sizes
differ by at most one row).  Per solve:

* zeta_0      local K0 abs-max, ``all_reduce(MAX)`` of one scalar (overlapped
              with the first sample draw, as on one GPU);
* sampled     every sampled entry has exactly one owner -- the rank whose slab
  blocks     holds its mode-1 index (core rows I_1 in the slab, mode-1 fiber
              rows in the slab, whole mode-k>=2 fibers whose decoded i_1 is in
              the slab).  The gather fills the owned entries, ``shard_pack``
              packs them (csrc/shard_xchg.cu), ONE all-gather of the padded
              packed segments moves each entry exactly once ((P-1)/P of
              E*N_blk received per rank), and ``shard_unpack`` rebuilds the
              compact blocks bit-identically to an unsharded gather.  Once for
              RTCUR-F; every iteration for RTCUR-R (the reference's regather,
              solver.py:315-322), prefetched behind the running iteration;
* the small CUR build, the error sums and the stop rule then run replicated
  and identically on every rank (deterministic kernels, identical inputs);
* full output K3 runs on the local slab; its two residual sums are
  ``all_reduce(SUM)``-ed.

One process per GPU (torchrun), backend "nccl" (NVLink / NVSwitch).  A "gloo"
group works too (exchange staged through host memory): the world-size-2 tests
run both ranks' engines on one device that way.
"""

from __future__ import annotations

import numpy as np

from .solver import SolverConfig, SolveResult, _solve, _Source
from .synth import slab_bounds
from .tensor import DeviceTensor

__all__ = ["rtcur_sharded", "full_output_sharded", "slab_bounds", "exchange_blocks"]


def _group(group):
    import torch.distributed as dist

    if group is not None:
        return group
    if not (dist.is_available() and dist.is_initialized()):
        raise RuntimeError("a sharded solve needs an initialised torch.distributed process group")
    return dist.group.WORLD


def group_size(group) -> int:
    import torch.distributed as dist

    return dist.get_world_size(group)


def group_rank(group) -> int:
    import torch.distributed as dist

    return dist.get_rank(group)


def _on_host(group) -> bool:
    """gloo groups move CUDA tensors through host memory."""
    import torch.distributed as dist

    return dist.get_backend(group) != "nccl"


def all_gather_host(t, group, device):
    """all-gather of a small tensor; returns the concatenation as a host tensor."""
    import torch
    import torch.distributed as dist

    world = group_size(group)
    src = t.cpu() if _on_host(group) else t.to(device)
    out = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out.cpu()


def all_reduce_max(v: float, group, device) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cpu" if _on_host(group) else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def exchange_blocks(eng, group):
    """Complete the compact sampled blocks of the staged sample from every rank's
    owned entries: plan -> pack -> all-gather -> unpack (csrc/shard_xchg.cu)."""
    import torch
    import torch.distributed as dist

    counts = eng.shard_plan()
    world = len(counts)
    maxc = max(1, max(counts))
    dtype = eng.torch_dtype
    bufs = getattr(eng, "_xchg", None)
    if bufs is None or bufs[0].numel() < maxc or bufs[1].numel() < world * maxc:
        cap = max(maxc, eng.nblk_total // max(world, 1) + 1)
        bufs = eng._xchg = (torch.empty(cap, dtype=dtype, device=eng.device),
                            torch.empty(world * cap, dtype=dtype, device=eng.device))
    send, recv = bufs[0][:maxc], bufs[1][:world * maxc]
    eng.shard_pack(send)
    if _on_host(group):
        torch.cuda.current_stream(eng.device).synchronize()
        rh = torch.empty(world * maxc, dtype=dtype)
        dist.all_gather_into_tensor(rh, send.cpu(), group=group)
        recv.copy_(rh)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)
    eng.shard_unpack(recv, maxc)


def rtcur_sharded(x_slab: DeviceTensor, global_shape, slab, cfg: SolverConfig, record_trace: bool = False,
                  group=None) -> SolveResult:
    """rtcur() on a mode-1-sharded tensor: ``x_slab`` is this rank's slab
    [lo, hi) of a ``global_shape`` tensor; ``group`` defaults to the world."""
    return _solve(_Source(x_slab, slab=tuple(slab), group=_group(group), global_shape=tuple(global_shape)), cfg,
                  record_trace)


def full_output_sharded(res: SolveResult, group=None):
    """K3 on the local slab: (L_slab, S_slab, global ||X - L - S|| / ||X||)."""
    import torch
    import torch.distributed as dist

    eng = res.cur._engine
    L, S, e2, x2 = eng.full_output(res.zeta_final)
    group = _group(group)
    t = torch.tensor([e2, x2], dtype=torch.float64, device="cpu" if _on_host(group) else eng.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    e2, x2 = float(t[0]), float(t[1])
    rel = float(np.sqrt(e2) / np.sqrt(x2)) if x2 > 0 else (0.0 if e2 == 0 else float("inf"))
    lo, hi = eng.slab
    shape = (hi - lo,) + tuple(eng.shape[1:])
    return DeviceTensor(L, shape), (DeviceTensor(S, shape) if S is not None else None), rel
