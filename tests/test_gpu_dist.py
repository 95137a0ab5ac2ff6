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
