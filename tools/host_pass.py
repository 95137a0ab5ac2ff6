"""Diagnostic: host time of each step of the solve loop's pass (draw, set_sample, gather,
iterate_async, iterate_wait), averaged over the iterations of a few solves.
usage: python tools/host_pass.py <config>"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200 import engine as E  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config, make_config_device  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if c <= 1:
    xf, _, _, bc = make_config(c)
    x = DeviceTensor(torch.from_numpy(xf).cuda(), bc.shape)
else:
    x, bc = make_config_device(c)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
T, N = {}, {}


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        N[name] = N.get(name, 0) + 1
        return r
    return w


for nm in ("set_sample", "gather", "iterate_async", "iterate_wait", "iterate_cancel"):
    setattr(E.Engine, nm, timed(nm, getattr(E.Engine, nm)))
for _ in range(3):
    res = rtcur(x, cfg)
    res = None
torch.cuda.synchronize()
T.clear()
N.clear()
t0 = time.perf_counter()
n = 5
for _ in range(n):
    res = None
    res = rtcur(x, cfg)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"config {c}: {1e3 * tot / n:.3f} ms/solve; per call (us): "
      + "  ".join(f"{k} {1e6 * T[k] / N[k]:.1f} (x{N[k] // n})" for k in T))
