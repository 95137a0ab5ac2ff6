"""Diagnostic: per-solve times of 30 back-to-back config-1 solves under the bench's
settings (PROFILE on one phase), with the garbage collector's pauses and the largest
host gaps of every slow solve.  usage: python tools/slow_solves.py [one|off] [gcoff]"""
import gc
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200 import solver as S  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "one"
xf, _, _, bc = make_config(1)
x = DeviceTensor(torch.from_numpy(xf).cuda(), bc.shape)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
if mode == "one":
    S.PROFILE, S.PROFILE_PHASES = True, ("error",)
if "gcoff" in sys.argv:
    gc.disable()
gct = [0.0, 0, 0.0]


def cb(phase, info):
    if phase == "start":
        gct[2] = time.perf_counter()
    else:
        gct[0] += time.perf_counter() - gct[2]
        gct[1] += 1


gc.callbacks.append(cb)
for _ in range(3):
    res = rtcur(x, cfg)
    res = None
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
per = []
for i in range(30):
    res = None
    gct[0], gct[1] = 0.0, 0
    S._TIMELINE = []
    t1 = time.perf_counter()
    res = rtcur(x, cfg)
    dt = 1e3 * (time.perf_counter() - t1)
    tl = S._TIMELINE
    S._TIMELINE = None
    per.append(round(dt, 2))
    if dt > 10.0:
        gaps = [(tl[j][0], tl[j][1], round(1e6 * (tl[j][2] - tl[j - 1][2]))) for j in range(1, len(tl))]
        print(f"  solve {i}: {dt:.2f} ms, gc {1e3 * gct[0]:.2f} ms in {gct[1]} collections; largest gaps "
              f"{sorted(gaps, key=lambda g: -g[2])[:4]}", flush=True)
ev1.record()
torch.cuda.synchronize()
print(f"mode {mode} {'gcoff' if 'gcoff' in sys.argv else ''}: {ev0.elapsed_time(ev1) / 30:.2f} ms/solve; per solve {per}")
