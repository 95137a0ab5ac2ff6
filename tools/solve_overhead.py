"""Diagnostic: per-solve wall/device time with and without per-phase profiling events."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200 import solver as S, synth
from paper_2108_10448_b200.tensor import DeviceTensor

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
x, _, _, bc = synth.make_config(cfgi)
X = DeviceTensor(torch.from_numpy(x).cuda(), bc.shape)
rows, cols = synth.baseline_sample_sizes(bc.shape, bc.ranks)
cfg = S.SolverConfig(ranks=bc.ranks, variant=bc.variant, eps=bc.eps, gamma=0.7, seed=bc.seed_solver + 1000,
                     row_sample_sizes=rows, col_sample_sizes=cols)
for _ in range(3):
    res = S.rtcur(X, cfg)
for prof in (False, True, False):
    S.PROFILE = prof
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); t0 = time.perf_counter(); it = 0; loop = 0.0
    for _ in range(10):
        res = S.rtcur(X, cfg)
        it += res.iterations
        loop += res.timings["loop"]
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"profile={prof}: {ms/10:.2f} ms/solve  {it/10:.1f} it/solve  {it/(ms/1e3):.1f} iters/s  loop {loop/10*1e3:.2f} ms  wall {(time.perf_counter()-t0)/10*1e3:.2f}")
S.PROFILE = False
# breakdown of the per-solve setup
import numpy as np
from paper_2108_10448_b200.fiber_cur import draw_sample_indices
from paper_2108_10448_b200.engine import acquire_engine
t = {}
src = S._Source(X)
t0 = time.perf_counter(); rng = np.random.default_rng(1); idx = draw_sample_indices(bc.shape, rows, cols, rng); t["draw"] = time.perf_counter() - t0
t0 = time.perf_counter(); eng = acquire_engine(bc.shape, bc.ranks, rows, cols, src.torch_dtype, slab=src.slab); t["acquire"] = time.perf_counter() - t0
t0 = time.perf_counter(); src.attach(eng); t["attach"] = time.perf_counter() - t0
t0 = time.perf_counter(); eng.set_sample(idx); t["set_sample"] = time.perf_counter() - t0
t0 = time.perf_counter(); src.load_blocks(eng, idx); torch.cuda.synchronize(); t["gather"] = time.perf_counter() - t0
t0 = time.perf_counter(); z = src.inf_norm(eng); t["absmax"] = time.perf_counter() - t0
print({k: round(v * 1e6, 1) for k, v in t.items()}, "us")
