# diagnostics: host-side cost of each step of the RTCUR-R loop (config 1)
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
from paper_2108_10448_b200.engine import Engine
from paper_2108_10448_b200.fiber_cur import draw_sample_indices
from paper_2108_10448_b200.synth import make_config, baseline_sample_sizes
xf, _, _, bc = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
dt = torch.float64 if bc.dtype == "f64" else torch.float32
x = DeviceTensor(torch.from_numpy(xf).to(dt).cuda(), bc.shape)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
for _ in range(3):
    rtcur(x, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter(); res = rtcur(x, cfg); torch.cuda.synchronize(); print("solve wall ms", (time.perf_counter() - t0) * 1e3, res.iterations)
eng = Engine(bc.shape, bc.ranks, rows, cols, dt)
eng.bind(x.flat)
rng = np.random.default_rng(bc.seed_solver)
zeta = eng.absmax()
acc = {k: 0.0 for k in ("draw", "set_sample", "gather", "launch", "wait")}
idx = draw_sample_indices(bc.shape, rows, cols, rng)
T0 = time.perf_counter()
for k in range(1, 26):
    t = time.perf_counter(); eng.set_sample(idx); acc["set_sample"] += time.perf_counter() - t
    t = time.perf_counter(); eng.gather(); acc["gather"] += time.perf_counter() - t
    zeta *= 0.7
    t = time.perf_counter(); eng.iterate_async(zeta, first=(k == 1)); acc["launch"] += time.perf_counter() - t
    t = time.perf_counter(); idx = draw_sample_indices(bc.shape, rows, cols, rng); acc["draw"] += time.perf_counter() - t
    t = time.perf_counter(); eng.iterate_wait(); acc["wait"] += time.perf_counter() - t
print("loop wall ms", (time.perf_counter() - T0) * 1e3)
print({k: round(v / 25 * 1e3, 3) for k, v in acc.items()}, "ms per iteration")
