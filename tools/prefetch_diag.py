"""Host timeline of the RTCUR-R loop (iterate_async / next-sample staging /
iterate_wait) to diagnose the side-stream prefetch.  One process per setting:
RTCUR_SIDE_PREFETCH=0|1 python tools/prefetch_diag.py 1"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import solver as S, synth  # noqa: E402
from paper_2108_10448_b200.engine import acquire_engine  # noqa: E402
from paper_2108_10448_b200.fiber_cur import draw_sample_indices  # noqa: E402
from paper_2108_10448_b200.tensor import DeviceTensor  # noqa: E402

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if cfgi <= 1:
    x, _, _, bc = synth.make_config(cfgi)
    X = DeviceTensor(torch.from_numpy(x).cuda(), bc.shape)
else:
    X, bc = synth.make_config_device(cfgi)
rows, cols = synth.baseline_sample_sizes(bc.shape, bc.ranks)
cfg = S.SolverConfig(ranks=bc.ranks, variant="R", eps=bc.eps, gamma=0.7, seed=bc.seed_solver, max_iters=100,
                     row_sample_sizes=rows, col_sample_sizes=cols)
for rep in range(3):
    res = S.rtcur(X, cfg)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
t0 = time.perf_counter()
for rep in range(3):
    res = None
    res = S.rtcur(X, cfg)
ev1.record()
torch.cuda.synchronize()
print(f"side={os.environ.get('RTCUR_SIDE_PREFETCH', '1')} config {cfgi}: {ev0.elapsed_time(ev1) / 3:.2f} ms/solve "
      f"host {1e3 * (time.perf_counter() - t0) / 3:.2f} ms, iters {res.iterations}")
# manual loop with host timestamps
src = S._Source(X)
rs, cs = cfg.resolve_sample_sizes(bc.shape)
rng = np.random.default_rng(cfg.seed)
res = None
eng = acquire_engine(bc.shape, bc.ranks, rs, cs, src.torch_dtype, slab=src.slab)
src.attach(eng)
idx = draw_sample_indices(bc.shape, rs, cs, rng)
eng.set_sample(idx)
src.load_blocks(eng, idx)
zeta = src.inf_norm(eng)
torch.cuda.synchronize()
rowsT = []
nxt = None
for k in range(1, 26):
    ta = time.perf_counter()
    zeta *= cfg.gamma
    eng.iterate_async(zeta, first=(k == 1))
    tb = time.perf_counter()
    nxt = draw_sample_indices(bc.shape, rs, cs, rng)
    tc = time.perf_counter()
    eng.set_sample(nxt)
    src.load_blocks(eng, nxt)
    td = time.perf_counter()
    eng.iterate_wait()
    te = time.perf_counter()
    rowsT.append((1e6 * (tb - ta), 1e6 * (tc - tb), 1e6 * (td - tc), 1e6 * (te - td), 1e6 * (te - ta)))
a = np.array(rowsT)
print("us per iteration  launch  draw  stage  wait  total")
print("median", np.round(np.median(a, 0), 1))
print("max   ", np.round(np.max(a, 0), 1))
for r in rowsT[:6]:
    print(np.round(r, 1))
