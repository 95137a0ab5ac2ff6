"""One fp32-storage parity solve (the test_gpu_parity.py case) for compute-sanitizer runs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_gaussian_tucker

shape, ranks = (40, 36, 30), (3, 3, 3)
xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=21, dtype=np.float32)
rows, cols = baseline_sample_sizes(shape, ranks)
kw = dict(eps=1e-5, variant="F", max_iters=3, seed=4, row_sample_sizes=rows, col_sample_sizes=cols)
res = rtcur(DeviceTensor(torch.from_numpy(xf).cuda(), shape), SolverConfig(ranks=ranks, **kw))
print(res.iterations, res.error_history)
