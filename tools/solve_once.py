"""One device-resident solve of a BASELINE config (for ncu captures): the
instance is generated on the device, then rtcur runs `--iters` iterations.

usage: python tools/solve_once.py --config 2 --iters 3 [--warm 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2108_10448_b200 import SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200.synth import CONFIGS, baseline_sample_sizes, make_config_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--warm", type=int, default=0)
a = ap.parse_args()
bc = CONFIGS[a.config]
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
x, _ = make_config_device(a.config)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, gamma=0.7, variant=bc.variant, max_iters=a.iters, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
for _ in range(a.warm + 1):
    res = rtcur(x, cfg)
torch.cuda.synchronize()
print("iterations", res.iterations, "err", res.error_history[-1])
