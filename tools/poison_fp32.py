"""Race / uninitialised-memory hunt: fill the caching allocator's memory with garbage,
free it, then solve the fp32-storage parity case in a fresh engine and compare the
iteration count with the fp64 oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import rtcur_oracle as orc
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_gaussian_tucker

variant = sys.argv[1] if len(sys.argv) > 1 else "F"
junk = torch.full((64 * 1024 * 1024,), 12345.678, dtype=torch.float64, device="cuda")
del junk
shape, ranks = (40, 36, 30), (3, 3, 3)
xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=21, dtype=np.float32)
rows, cols = baseline_sample_sizes(shape, ranks)
kw = dict(eps=1e-5, variant=variant, max_iters=100, seed=4, row_sample_sizes=rows, col_sample_sizes=cols)
ref = orc.solve(xf.astype(np.float64), shape, ranks, **kw)
dev = DeviceTensor(torch.from_numpy(xf).cuda(), shape)
res = rtcur(dev, SolverConfig(ranks=ranks, **kw))
ok = res.iterations == ref.iterations
print("OK" if ok else "BAD", res.iterations, ref.iterations,
      next((k for k, (a, b) in enumerate(zip(res.error_history, ref.error_history)) if abs(a - b) > 1e-8), None))
