"""Multi-rank host logic on CPU (gloo, world size 2): mode-1 slab ownership of
the sampled blocks + sum all-reduce reproduces the full gather bit-exactly
(SURVEY §8(e)).  The per-rank gather here is a numpy emulation of the device
ownership rule of k_gather (entry kept iff its mode-1 index is in the rank's
slab); the device kernel itself is checked against the same rule on one GPU in
tests/test_gpu_dist.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rtcur_oracle as orc
from paper_2108_10448_b200.fiber_cur import draw_sample_indices
from paper_2108_10448_b200.synth import slab_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def owned_blocks(x_flat, shape, idx, lo, hi):
    """Compact blocks [core | C_1 | .. | C_n] with entries outside mode-1 slab [lo, hi) zeroed."""
    arr = x_flat.reshape(shape, order="F")
    core = orc.core_block(arr, idx.rows).reshape(-1, order="F").copy()
    i1_core = np.broadcast_to((idx.rows[0] - 1).reshape((-1,) + (1,) * (len(shape) - 1)),
                              tuple(r.size for r in idx.rows)).reshape(-1, order="F")
    core[(i1_core < lo) | (i1_core >= hi)] = 0.0
    parts = [core]
    for k, cols in enumerate(idx.cols, start=1):
        fib = orc.gather_fibers(x_flat, shape, k, cols).copy()
        if k == 1:
            fib[:lo, :] = 0.0
            fib[hi:, :] = 0.0
        else:
            i1 = orc.decode_fiber_columns(shape, k, cols)[0] - 1
            fib[:, (i1 < lo) | (i1 >= hi)] = 0.0
        parts.append(fib.reshape(-1, order="F"))
    return np.concatenate(parts)


def _worker(rank, world, port, shape, ranks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(int(np.prod(shape)))
    rows = tuple(min(d, 4) for d in shape)
    total = int(np.prod(shape))
    cols = tuple(min(total // d, 9) for d in shape)
    idx = draw_sample_indices(shape, rows, cols, np.random.default_rng(11))
    lo, hi = slab_bounds(shape[0], world, rank)
    mine = torch.from_numpy(owned_blocks(x, shape, idx, lo, hi))
    dist.all_reduce(mine, op=dist.ReduceOp.SUM)
    # zeta_0: max all-reduce of the slab abs-max
    zt = torch.tensor([float(np.max(np.abs(x.reshape(shape, order="F")[lo:hi])))], dtype=torch.float64)
    dist.all_reduce(zt, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = owned_blocks(x, shape, idx, 0, shape[0])
        q.put((bool(np.array_equal(mine.numpy(), full)), float(zt.item()) == float(np.max(np.abs(x)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(7, 5, 4), (9, 4, 3, 2)])
def test_slab_allreduce_reproduces_full_gather(shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, None, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok_blocks, ok_zeta = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok_blocks and ok_zeta


def test_slab_bounds_partition():
    for d1 in (1, 7, 220, 1200):
        for world in (1, 2, 3, 8):
            if world > d1:
                continue
            b = [slab_bounds(d1, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == d1
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in b]
            assert max(sizes) - min(sizes) <= 1
    assert [h - l for l, h in (slab_bounds(220, 8, r) for r in range(8))].count(28) == 4
