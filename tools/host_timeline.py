"""Diagnostic: host-side time breakdown of one RTCUR solve loop (config 1)."""
import time, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200 import solver as S
from paper_2108_10448_b200 import synth
from paper_2108_10448_b200.fiber_cur import draw_sample_indices
from paper_2108_10448_b200.tensor import DeviceTensor

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
x, _, _, bc = synth.make_config(cfgi)
X = DeviceTensor(torch.from_numpy(x).cuda(), bc.shape)
rows, cols = synth.baseline_sample_sizes(bc.shape, bc.ranks)
cfg = S.SolverConfig(ranks=bc.ranks, variant=bc.variant, eps=bc.eps, seed=bc.seed_solver,
                     row_sample_sizes=rows, col_sample_sizes=cols)
for _ in range(3):
    S.rtcur(X, cfg)
torch.cuda.synchronize()
# manual loop mirroring solver._solve with host timestamps
src = S._Source(X)
shape = src.shape
rng = np.random.default_rng(cfg.seed)
rs, cs = cfg.resolve_sample_sizes(shape)
idx = draw_sample_indices(shape, rs, cs, rng)
eng = S.acquire_engine(shape, cfg.ranks, rs, cs, src.torch_dtype, slab=src.slab)
src.attach(eng)
eng.set_sample(idx); src.load_blocks(eng, idx)
zeta = src.inf_norm(eng)
torch.cuda.synchronize()
acc = {k: 0.0 for k in ("set_sample", "load", "launch", "draw", "wait", "py")}
nxt = None
t_begin = time.perf_counter()
K = 25
for k in range(1, K + 1):
    t0 = time.perf_counter()
    if cfg.variant == "R" and k >= 2:
        idx = nxt
        eng.set_sample(idx); t1 = time.perf_counter(); acc["set_sample"] += t1 - t0
        src.load_blocks(eng, idx); t0 = time.perf_counter(); acc["load"] += t0 - t1
    zeta *= cfg.gamma
    eng.iterate_async(zeta, first=(k == 1)); t1 = time.perf_counter(); acc["launch"] += t1 - t0
    if cfg.variant == "R":
        nxt = draw_sample_indices(shape, rs, cs, rng)
    t2 = time.perf_counter(); acc["draw"] += t2 - t1
    e2, x2, fl = eng.iterate_wait(); t3 = time.perf_counter(); acc["wait"] += t3 - t2
    err = S._error_from_sums(e2, x2); acc["py"] += time.perf_counter() - t3
tot = time.perf_counter() - t_begin
print(f"config{cfgi}: {K} iters {tot*1e3:.2f} ms  per-iter {tot/K*1e6:.1f} us")
for k, v in acc.items():
    print(f"  {k:10s} {v/K*1e6:8.1f} us/iter")
