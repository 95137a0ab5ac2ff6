"""Uninitialised-memory hunt: poison the allocator, solve the fp32 parity case with
record_trace and compare iteration 1's sparse/low-rank blocks and SVD with the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import rtcur_oracle as orc
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_gaussian_tucker

junk = torch.full((64 * 1024 * 1024,), 12345.678, dtype=torch.float64, device="cuda")
del junk
shape, ranks = (40, 36, 30), (3, 3, 3)
xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=21, dtype=np.float32)
rows, cols = baseline_sample_sizes(shape, ranks)
kw = dict(eps=1e-5, variant="F", max_iters=2, seed=4, row_sample_sizes=rows, col_sample_sizes=cols)
ref = orc.solve(xf.astype(np.float64), shape, ranks, record_trace=True, **kw)
res = rtcur(DeviceTensor(torch.from_numpy(xf).cuda(), shape), SolverConfig(ranks=ranks, **kw), record_trace=True)
print("err", res.error_history, ref.error_history)
t, r = res.trace[0], ref.trace[0]
rk = list(r.keys()) if isinstance(r, dict) else dir(r)
print("oracle trace keys", rk)
for key in ("s_core", "l_core"):
    a = np.asarray(t[key]).reshape(-1, order="F"); b = np.asarray(r[key]).reshape(-1, order="F")
    print(key, np.abs(a - b).max())
for m in range(3):
    for key in ("s_fibers", "l_fibers"):
        a = np.asarray(t[key][m]); b = np.asarray(r[key][m])
        d = np.abs(a - b)
        print(m, key, d.max(), np.unravel_index(d.argmax(), d.shape), a.shape)
for m in range(3):
    print("sv", m, res.cur.intersections[m].singular_values, ref.cur.intersections[m].singular_values)
