"""Diagnostic: per-step wall time of bench.py's e2e loop (config 1), split into
H2D, solve and result export, to see where the end-to-end variance comes from."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200 import solver as S, synth
from paper_2108_10448_b200.tensor import DeviceTensor

x, _, _, bc = synth.make_config(1)
rows, cols = synth.baseline_sample_sizes(bc.shape, bc.ranks)
cfg = S.SolverConfig(ranks=bc.ranks, variant=bc.variant, eps=bc.eps, gamma=0.7, seed=bc.seed_solver,
                     row_sample_sizes=rows, col_sample_sizes=cols, max_iters=100)
pinned = torch.from_numpy(x).pin_memory()
buf = torch.empty(pinned.numel(), dtype=torch.float64, device="cuda")
res = None
for rep in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    buf.copy_(pinned, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    res = None
    res = S.rtcur(DeviceTensor(buf, bc.shape), cfg); t2 = time.perf_counter()
    a = (res.sparse.core, res.sparse.fibers, res.cur.core, res.cur.fibers, res.cur.intersections, res.cur.factors)
    t3 = time.perf_counter()
    print(f"rep {rep}: h2d {1e3*(t1-t0):.1f}  solve {1e3*(t2-t1):.1f}  export {1e3*(t3-t2):.1f}  total {1e3*(t3-t0):.1f} ms", flush=True)
