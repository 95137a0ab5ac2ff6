"""Small solves for compute-sanitizer runs (memcheck / initcheck / racecheck /
synccheck): BASELINE config-0 geometry (100^3, ranks 3, BASELINE sample sizes)
for RTCUR-F and RTCUR-R, fp64 and fp32 storage, plus K3 and the sharded
pack/unpack of two virtual ranks.  Kept short (a few iterations): the
sanitizer serialises and instruments every launch.

usage: compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_solve.py [--iters 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_10448_b200 import DeviceTensor, SolverConfig, full_output, rtcur  # noqa: E402
from paper_2108_10448_b200.engine import Engine  # noqa: E402
from paper_2108_10448_b200.fiber_cur import draw_sample_indices  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config, slab_bounds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
xf, _, _, bc = make_config(0)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
for dt in (torch.float64, torch.float32):
    x = DeviceTensor(torch.from_numpy(xf).to(dt).cuda(), bc.shape)
    for variant in ("F", "R"):
        cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=variant, max_iters=a.iters, seed=0,
                           row_sample_sizes=rows, col_sample_sizes=cols)
        res = rtcur(x, cfg)
        L, S, rel = full_output(res, x)
        _ = (res.sparse.core, res.cur.factors)
        print(dt, variant, res.iterations, res.error_history[-1], rel, flush=True)
        del res, L, S
# sharded exchange kernels (two virtual ranks, no collective)
x = torch.from_numpy(xf).cuda()
xr = x.reshape(tuple(reversed(bc.shape)))
idx = draw_sample_indices(bc.shape, rows, cols, np.random.default_rng(1))
bounds = [slab_bounds(bc.shape[0], 2, r)[0] for r in range(2)] + [bc.shape[0]]
engs = []
for r in range(2):
    e = Engine(bc.shape, bc.ranks, rows, cols, torch.float64, slab=(bounds[r], bounds[r + 1]))
    e._part = xr[..., bounds[r]:bounds[r + 1]].contiguous().reshape(-1)
    e.bind(e._part)
    e.set_shards(2, r, bounds)
    e.set_sample(idx)
    e.gather()
    engs.append((e, e.shard_plan()))
stride = max(engs[0][1])
recv = torch.zeros(2 * stride, dtype=torch.float64, device="cuda")
for r, (e, _) in enumerate(engs):
    e.shard_pack(recv[r * stride:(r + 1) * stride])
for e, _ in engs:
    e.shard_unpack(recv, stride)
torch.cuda.synchronize()
print("shard exchange ok", flush=True)
