"""Repeat the fp32-storage parity case (test_gpu_parity.py) N times in one process and
count iteration-count mismatches against the fp64 oracle (race hunting)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import rtcur_oracle as orc
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_gaussian_tucker

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
variant = sys.argv[2] if len(sys.argv) > 2 else "F"
shape, ranks = (40, 36, 30), (3, 3, 3)
xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=21, dtype=np.float32)
rows, cols = baseline_sample_sizes(shape, ranks)
kw = dict(eps=1e-5, variant=variant, max_iters=100, seed=4, row_sample_sizes=rows, col_sample_sizes=cols)
ref = orc.solve(xf.astype(np.float64), shape, ranks, **kw)
dev = DeviceTensor(torch.from_numpy(xf).cuda(), shape)
bad = 0
hist0 = None
for i in range(n):
    res = rtcur(dev, SolverConfig(ranks=ranks, **kw))
    if res.iterations != ref.iterations:
        bad += 1
        print("run", i, "iterations", res.iterations, "vs", ref.iterations, "first err diff at",
              next((k for k, (a, b) in enumerate(zip(res.error_history, ref.error_history)) if abs(a - b) > 1e-8), None))
    if hist0 is None:
        hist0 = list(res.error_history)
    elif list(res.error_history) != hist0:
        print("run", i, "history differs from run 0 (nondeterminism)")
print("bad", bad, "of", n)
