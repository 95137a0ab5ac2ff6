"""Sharding on one GPU: the device gather's slab ownership, the slab-independent
instance generator, and the sharded solve path through a 1-rank NCCL group."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200.engine import Engine  # noqa: E402
from paper_2108_10448_b200.fiber_cur import draw_sample_indices  # noqa: E402
from paper_2108_10448_b200.synth import (baseline_sample_sizes, make_gaussian_tucker_device,  # noqa: E402
                                         slab_bounds)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_virtual_slabs_sum_to_full_gather(dtype):
    shape, ranks = (23, 17, 11), (2, 2, 2)
    x = torch.randn(int(np.prod(shape)), dtype=torch.float64, device="cuda").to(dtype)
    rows, cols = baseline_sample_sizes(shape, ranks)
    idx = draw_sample_indices(shape, rows, cols, np.random.default_rng(1))
    full = Engine(shape, ranks, rows, cols, dtype)
    full.bind(x)
    full.set_sample(idx)
    full.gather()
    ref = full.xblocks().clone()
    xr = x.reshape(tuple(reversed(shape)))
    for world in (2, 3, 5):
        acc = torch.zeros_like(ref)
        amax = 0.0
        for r in range(world):
            lo, hi = slab_bounds(shape[0], world, r)
            part = xr[..., lo:hi].contiguous().reshape(-1)
            e = Engine(shape, ranks, rows, cols, dtype, slab=(lo, hi))
            e.bind(part)
            e.set_sample(idx)
            e.gather()
            acc += e.xblocks()
            amax = max(amax, e.absmax())
        assert torch.equal(acc, ref), world
        assert amax == float(x.abs().max())


def test_generator_is_slab_independent():
    shape, ranks = (30, 12, 9, 5), (3, 2, 2, 2)
    full, mu = make_gaussian_tucker_device(shape, ranks, 0.2, 10.0, seed=5, dtype=torch.float32)
    fr = full.flat.reshape(tuple(reversed(shape)))
    for world in (2, 4):
        for r in range(world):
            lo, hi = slab_bounds(shape[0], world, r)
            part, _ = make_gaussian_tucker_device(shape, ranks, 0.2, 10.0, seed=5, dtype=torch.float32,
                                                  slab=(lo, hi), mu=mu)
            assert torch.equal(part.flat.reshape(tuple(reversed(part.shape))), fr[..., lo:hi])
    # outlier density ~ alpha
    low, _ = make_gaussian_tucker_device(shape, ranks, 0.0, 10.0, seed=5, dtype=torch.float32, mu=mu)
    frac = float((full.flat != low.flat).double().mean())
    assert 0.15 < frac < 0.25


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_solve_single_rank_matches_plain():
    import torch.distributed as dist

    from paper_2108_10448_b200.dist import full_output_sharded, rtcur_sharded

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_port()))
        dist.init_process_group("nccl", rank=0, world_size=1)
    shape, ranks = (26, 20, 18), (2, 2, 2)
    x, _ = make_gaussian_tucker_device(shape, ranks, 0.15, 10.0, seed=9, dtype=torch.float64)
    rows, cols = baseline_sample_sizes(shape, ranks)
    for variant in ("F", "R"):
        cfg = SolverConfig(ranks=ranks, variant=variant, max_iters=60, seed=2, row_sample_sizes=rows,
                           col_sample_sizes=cols)
        a = rtcur(x, cfg)
        b = rtcur_sharded(x, shape, (0, shape[0]), cfg)
        assert a.error_history == b.error_history
        assert np.array_equal(a.sparse.core, b.sparse.core)
        _, _, rel = full_output_sharded(b)
        assert rel < 1e-3
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("shape", [(23, 17, 11), (13, 9, 7, 5)])
def test_virtual_ranks_pack_unpack_reproduce_full_gather(dtype, shape):
    """csrc/shard_xchg.cu without a collective: every virtual rank's engine packs
    its owned entries; the concatenated padded segments (what the all-gather
    delivers) unpack into every rank's blocks bit-identically to the unsharded
    gather, and the counts add up to N_blk (each entry sent once)."""
    ranks = (2,) * len(shape)
    x = torch.randn(int(np.prod(shape)), dtype=torch.float64, device="cuda").to(dtype)
    rows, cols = baseline_sample_sizes(shape, ranks)
    xr = x.reshape(tuple(reversed(shape)))
    for seed in (1, 2):
        idx = draw_sample_indices(shape, rows, cols, np.random.default_rng(seed))
        full = Engine(shape, ranks, rows, cols, dtype)
        full.bind(x)
        full.set_sample(idx)
        full.gather()
        ref = full.xblocks().clone()
        for world in (2, 3, 5):
            bounds = [slab_bounds(shape[0], world, r)[0] for r in range(world)] + [shape[0]]
            engs, counts = [], None
            for r in range(world):
                lo, hi = bounds[r], bounds[r + 1]
                e = Engine(shape, ranks, rows, cols, dtype, slab=(lo, hi))
                e._part = xr[..., lo:hi].contiguous().reshape(-1)
                e.bind(e._part)
                e.set_shards(world, r, bounds)
                e.set_sample(idx)
                e.gather()
                c = e.shard_plan()
                assert counts is None or c == counts
                counts = c
                engs.append(e)
            assert sum(counts) == sum(p * q for p, q in full.block_shapes)   # each entry sent once
            stride = max(counts)
            recv = torch.full((world * stride,), float("nan"), dtype=dtype, device="cuda")
            for r, e in enumerate(engs):
                e.shard_pack(recv[r * stride:(r + 1) * stride])
            for e in engs:
                e.shard_unpack(recv, stride)
                got = e.xblocks()
                for b, (p, q) in enumerate(full.block_shapes):
                    o = full.block_offsets[b]
                    assert torch.equal(got[o:o + p * q], ref[o:o + p * q]), (world, b)


def _sharded_worker(rank, world, port, shape, ranks, variant, dtype_name, q):
    import torch.distributed as dist

    from paper_2108_10448_b200.dist import full_output_sharded, rtcur_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dtype = getattr(torch, dtype_name)
    x, _ = make_gaussian_tucker_device(shape, ranks, 0.2, 10.0, seed=21, dtype=dtype)
    lo, hi = slab_bounds(shape[0], world, rank)
    part = x.flat.reshape(tuple(reversed(shape)))[..., lo:hi].contiguous().reshape(-1)
    rows, cols = baseline_sample_sizes(shape, ranks)
    cfg = SolverConfig(ranks=ranks, variant=variant, max_iters=80, seed=4, row_sample_sizes=rows,
                       col_sample_sizes=cols)
    res = rtcur_sharded(DeviceTensor(part, (hi - lo,) + tuple(shape[1:])), shape, (lo, hi), cfg)
    L, S, rel = full_output_sharded(res)
    out = {"err": list(res.error_history), "it": res.iterations, "conv": res.converged,
           "s_core": np.asarray(res.sparse.core), "s_fib": [np.asarray(f) for f in res.sparse.fibers],
           "L": L.flat.cpu().numpy(), "S": S.flat.cpu().numpy(), "rel": rel, "slab": (lo, hi),
           "diag": list(res.diagnostics)}
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant,shape,ranks,dtype_name", [
    ("F", (26, 20, 18), (2, 2, 2), "float64"),
    ("R", (26, 20, 18), (2, 2, 2), "float64"),
    ("R", (15, 12, 10, 9), (2, 2, 2, 2), "float32"),
])
def test_world2_sharded_solve_matches_single_gpu(variant, shape, ranks, dtype_name):
    """rtcur_sharded at world size 2 (two processes, gloo, both engines on cuda:0;
    no kernel waits on another rank's kernel) reproduces the single-GPU solve
    bit for bit: error history, iteration count, S support and values,
    deficiency flags; K3 on the slabs concatenates to the single-GPU L and S."""
    import torch.multiprocessing as mp

    from paper_2108_10448_b200.full import full_output

    dtype = getattr(torch, dtype_name)
    x, _ = make_gaussian_tucker_device(shape, ranks, 0.2, 10.0, seed=21, dtype=dtype)
    rows, cols = baseline_sample_sizes(shape, ranks)
    cfg = SolverConfig(ranks=ranks, variant=variant, max_iters=80, seed=4, row_sample_sizes=rows,
                       col_sample_sizes=cols)
    ref = rtcur(x, cfg)
    L, S, rel = full_output(ref, x)
    Lr = L.flat.reshape(tuple(reversed(shape))).cpu().numpy()
    Sr = S.flat.reshape(tuple(reversed(shape))).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, shape, ranks, variant, dtype_name, q))
             for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, o in outs.items():
        assert o["err"] == list(ref.error_history), rank
        assert o["it"] == ref.iterations and o["conv"] == ref.converged
        assert o["diag"] == list(ref.diagnostics)
        assert np.array_equal(o["s_core"], np.asarray(ref.sparse.core))
        for a, b in zip(o["s_fib"], ref.sparse.fibers):
            assert np.array_equal(a, np.asarray(b))
        lo, hi = o["slab"]
        w = hi - lo
        assert np.array_equal(o["L"].reshape(Lr[..., lo:hi].shape), Lr[..., lo:hi])
        assert np.array_equal(o["S"].reshape(Sr[..., lo:hi].shape), Sr[..., lo:hi])
        assert abs(o["rel"] - rel) <= 1e-12 * max(rel, 1e-300) + 1e-15
        assert w > 0
