"""Diagnostic: what the per-iteration host round trip costs.  Fixed 25 iterations (eps=0)
with and without RTCUR_NOWAIT_DIAG=1 (iterate_wait returns without a host sync).
usage: [RTCUR_NOWAIT_DIAG=1] python tools/nowait_diag.py <config>"""
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
cfg = SolverConfig(ranks=bc.ranks, eps=1e-300, variant=bc.variant, max_iters=25, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
for _ in range(3):
    res = rtcur(x, cfg)
    res = None
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
t0 = time.perf_counter()
for _ in range(5):
    res = None
    res = rtcur(x, cfg)
ev1.record()
torch.cuda.synchronize()
print(f"config {c} nowait={os.environ.get('RTCUR_NOWAIT_DIAG', '0')} side={os.environ.get('RTCUR_SIDE_PREFETCH', '0')}: "
      f"{ev0.elapsed_time(ev1) / 5:.3f} ms/solve (25 iterations), host {1e3 * (time.perf_counter() - t0) / 5:.3f}")
