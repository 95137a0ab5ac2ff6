"""Multi-rank host logic on CPU (gloo, world sizes 2 and 3): mode-1 slab
ownership of the sampled blocks and the pack -> all-gather -> unpack exchange
(csrc/shard_xchg.cu) reproduce the full gather bit-exactly.

``plan`` / ``pack`` / ``unpack`` below restate the device protocol in numpy:
per block a row band x column set per rank (core: rows I_1 in the slab, all
columns; mode-1 fibers: rows [lo, hi), all columns; mode-k>=2 fibers: all rows
of the columns whose decoded i_1 lies in the slab, in increasing column
order), packed block after block, one column's band contiguous.  The device
kernels are checked against the unsharded gather on the GPU
(tests/test_gpu_dist.py, including a world-2 solve on one device)."""

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


def full_blocks(x_flat, shape, idx):
    arr = x_flat.reshape(shape, order="F")
    blocks = [orc.core_block(arr, idx.rows).reshape(len(idx.rows[0]), -1, order="F")]
    blocks += [orc.gather_fibers(x_flat, shape, k, c) for k, c in enumerate(idx.cols, start=1)]
    return blocks


def plan(shape, idx, bounds):
    """[rank][block] -> (row band r0:r1, column list) as shard_plan builds it."""
    world = len(bounds) - 1
    rows0 = idx.rows[0] - 1
    q_core = int(np.prod([r.size for r in idx.rows[1:]]))
    out = []
    for p in range(world):
        lo, hi = bounds[p], bounds[p + 1]
        r0, r1 = np.searchsorted(rows0, lo), np.searchsorted(rows0, hi)
        segs = [(r0, r1, np.arange(q_core) if r1 > r0 else np.arange(0))]
        segs.append((lo, hi, np.arange(idx.cols[0].size) if hi > lo else np.arange(0)))
        for k in range(2, len(shape) + 1):
            i1 = (idx.cols[k - 1] - 1) % shape[0]
            segs.append((0, shape[k - 1], np.nonzero((i1 >= lo) & (i1 < hi))[0]))
        out.append(segs)
    return out


def pack(blocks, segs):
    return np.concatenate([blocks[b][r0:r1, cols].reshape(-1, order="F") for b, (r0, r1, cols) in enumerate(segs)])


def unpack(recv, stride, pl, blocks_out):
    for p, segs in enumerate(pl):
        o = p * stride
        for b, (r0, r1, cols) in enumerate(segs):
            n = (r1 - r0) * cols.size
            blocks_out[b][r0:r1, cols] = recv[o:o + n].reshape((r1 - r0, cols.size), order="F")
            o += n


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
    bounds = [slab_bounds(shape[0], world, p)[0] for p in range(world)] + [shape[0]]
    lo, hi = bounds[rank], bounds[rank + 1]
    pl = plan(shape, idx, bounds)
    counts = [sum((r1 - r0) * c.size for r0, r1, c in segs) for segs in pl]
    stride = max(counts)
    # this rank's gather: the full blocks stand in (only the owned entries are packed)
    owned = [b.copy() for b in full_blocks(x, shape, idx)]
    send = np.zeros(stride)
    mine = pack(owned, pl[rank])
    send[:mine.size] = mine
    recv = torch.empty(world * stride, dtype=torch.float64)
    dist.all_gather_into_tensor(recv, torch.from_numpy(send))
    got = [np.full_like(b, np.nan) for b in owned]
    unpack(recv.numpy(), stride, pl, got)
    # zeta_0: max all-reduce of the slab abs-max
    zt = torch.tensor([float(np.max(np.abs(x.reshape(shape, order="F")[lo:hi])))], dtype=torch.float64)
    dist.all_reduce(zt, op=dist.ReduceOp.MAX)
    full = full_blocks(x, shape, idx)
    ok = all(np.array_equal(a, b) for a, b in zip(got, full))
    # each entry is sent exactly once: the counts add up to N_blk
    once = sum(counts) == sum(b.size for b in full)
    # ownership is by the mode-1 index: a rank's packed entries all come from its slab
    arr = x.reshape(shape, order="F")
    slab_vals = set(arr[lo:hi].reshape(-1).tolist())
    local = all(v in slab_vals for v in mine.tolist())
    q.put((rank, ok, once, local, float(zt.item()) == float(np.max(np.abs(x)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("shape", [(7, 5, 4), (9, 4, 3, 2)])
def test_packed_allgather_reproduces_full_gather(shape, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, None, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, once, local, ok_zeta in res:
        assert ok and once and local and ok_zeta, rank


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
