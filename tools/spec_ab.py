"""A/B of the speculative pipeline / side prefetch: device-resident solves of a BASELINE
config, events around 5 solves after 3 warm-ups.  Settings come from the environment
(RTCUR_SPECULATE, RTCUR_SPEC, RTCUR_SIDE_PREFETCH).  usage: python tools/spec_ab.py <config>"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
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
for _ in range(3):
    res = rtcur(x, cfg)
    h = res.error_history
    res = None
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
t0 = time.perf_counter()
n = 5
for _ in range(n):
    res = None
    res = rtcur(x, cfg)
ev1.record()
torch.cuda.synchronize()
env = " ".join(f"{k}={os.environ[k]}" for k in ("RTCUR_SPECULATE", "RTCUR_SPEC", "RTCUR_SIDE_PREFETCH") if k in os.environ)
print(f"config {c} [{env}]: {ev0.elapsed_time(ev1) / n:.3f} ms/solve, {res.iterations} iterations "
      f"({res.iterations * n / ev0.elapsed_time(ev1) * 1e3:.0f} iters/s), host {1e3 * (time.perf_counter() - t0) / n:.3f} ms, "
      f"err {res.error_history[-1]:.3e} converged {res.converged}")
