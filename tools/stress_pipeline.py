"""Stress test of the iteration pipeline (speculation, held-back tail, shadow iterate, side
staging): random small problems, F and R, 2-4 modes, fp64 / fp32; every solve is run with the
pipelined loop and with the one-at-a-time loop and the two results must be identical (error
history, iteration count, sparse support and values, sigma).  Repeated solves reuse pooled
engines, so launch-shape rotation, cancels and resets are exercised too.
usage: python tools/stress_pipeline.py [n_problems] [seed]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200 import solver as S  # noqa: E402
from paper_2108_10448_b200.synth import make_gaussian_tucker  # noqa: E402

n_prob = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
solved = iters_total = stops = 0
t0 = time.time()
for p in range(n_prob):
    n = int(rng.integers(2, 5))
    dims = tuple(int(v) for v in rng.integers(12, 41 if n <= 3 else 25, size=n))
    ranks = tuple(int(v) for v in rng.integers(1, 4, size=n))
    alpha = float(rng.choice([0.0, 0.05, 0.15, 0.3]))
    xf, _, _ = make_gaussian_tucker(dims, ranks, alpha, 10.0, seed=int(rng.integers(1 << 30)))
    rows = tuple(int(min(d, max(r + 1, rng.integers(r + 1, d + 1)))) for d, r in zip(dims, ranks))
    rest = [int(np.prod(dims)) // d for d in dims]
    cols = tuple(int(min(q, max(r + 2, rng.integers(r + 2, min(q, 400) + 1)))) for q, r in zip(rest, ranks))
    variant = str(rng.choice(["F", "R"]))
    max_iters = int(rng.choice([1, 2, 3, 7, 40]))
    dt = torch.float64 if rng.random() < 0.6 else torch.float32
    cfg = SolverConfig(ranks=ranks, eps=float(rng.choice([1e-5, 1e-3])), variant=variant, max_iters=max_iters,
                       seed=int(rng.integers(1 << 30)), row_sample_sizes=rows, col_sample_sizes=cols)
    x = DeviceTensor.from_host(xf.reshape(dims, order="F").astype(np.float64 if dt == torch.float64 else np.float32))
    out = []
    try:
        for spec in (True, False, True):
            S.SPECULATE = spec
            res = rtcur(x, cfg)
            out.append((res.iterations, res.converged, tuple(res.error_history),
                        np.array(res.sparse.core).copy(), [np.array(f).copy() for f in res.sparse.fibers],
                        [np.array(t.singular_values).copy() for t in res.cur.intersections]))
            del res
    except ValueError as exc:   # (e.g. non-finite input of a degenerate draw: the same on both paths)
        print(f"problem {p}: {type(exc).__name__}: {str(exc)[:80]}")
        continue
    finally:
        S.SPECULATE = True
    solved += 1
    iters_total += out[0][0]
    stops += int(out[0][1])
    ok = True
    for other in out[1:]:
        ok &= out[0][:3] == other[:3] and np.array_equal(out[0][3], other[3])
        ok &= all(np.array_equal(a, b) for a, b in zip(out[0][4], other[4]))
        ok &= all(np.array_equal(a, b) for a, b in zip(out[0][5], other[5]))
    if not ok:
        bad += 1
        print(f"MISMATCH problem {p}: dims {dims} ranks {ranks} variant {variant} max_iters {max_iters} dtype {dt} "
              f"iters {[o[0] for o in out]}")
print(f"{n_prob} problems, {solved} compared ({iters_total} iterations, {stops} converged), {bad} mismatches, {time.time() - t0:.1f} s")
sys.exit(1 if bad else 0)
