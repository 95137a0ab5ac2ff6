"""Diagnostic: phase-transition sweep throughput (trials/s) vs concurrent workers."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200.sweeps import run_phase_transition

kw = dict(alphas=(0.1, 0.2, 0.3), upsilons=(2.0, 3.0), trials=8, n=3, d=60, r=3, variant="F", max_iters=150)
run_phase_transition(workers=4, **dict(kw, trials=2))   # warm-up (engine pools, kernels)
for w in (1, 2, 4, 8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = run_phase_transition(workers=w, **kw)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    n = len(kw["alphas"]) * len(kw["upsilons"]) * kw["trials"]
    print(f"workers={w}: {n} trials in {dt:.2f}s = {n/dt:.1f} trials/s  successes={g.successes}")
