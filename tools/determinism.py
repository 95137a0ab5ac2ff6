"""Run-to-run determinism of the pipelined solve at a BASELINE config: N solves on the pooled
engine, error history / iteration count / sparse-core digest must be identical every time.
usage: python tools/determinism.py <config> [n]"""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config, make_config_device  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if c <= 1:
    xf, _, _, bc = make_config(c)
    x = DeviceTensor(torch.from_numpy(xf).cuda(), bc.shape)
else:
    x, bc = make_config_device(c)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
seen = set()
for i in range(n):
    res = rtcur(x, cfg)
    dig = hashlib.sha256(np.ascontiguousarray(res.sparse.core).tobytes()).hexdigest()[:16]
    seen.add((res.iterations, tuple(res.error_history), dig))
    del res
print(f"config {c}: {n} solves, {len(seen)} distinct result(s)")
sys.exit(0 if len(seen) == 1 else 1)
