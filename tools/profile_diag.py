"""Time config-1 solves with the bench's profiling settings (PROFILE on one phase /
all phases / off) to find host gaps.  python tools/profile_diag.py [config]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200 import solver as S  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config, make_config_device  # noqa: E402
from paper_2108_10448_b200 import engine as E  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if c <= 1:
    xf, _, _, bc = make_config(c)
    x = DeviceTensor(torch.from_numpy(xf).cuda(), bc.shape)
else:
    x, bc = make_config_device(c)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
import gc  # noqa: E402

mode = os.environ.get("DIAG_GC", "")
if mode == "freeze":
    gc.freeze()
elif mode == "off":
    gc.disable()
print("gc mode:", mode or "default", "tracked objects:", len(gc.get_objects()), flush=True)
for label, prof, phases in (("off", False, None), ("one-phase", True, ("error",)), ("all", True, None),
                            ("off-again", False, None)):
    S.PROFILE, S.PROFILE_PHASES = prof, phases
    res = rtcur(x, cfg)
    res = None
    torch.cuda.synchronize()
    c0 = E.CREATED[0]
    t0 = time.perf_counter()
    per = []
    for _ in range(3):
        res = None
        S._TIMELINE = []
        t1 = time.perf_counter()
        res = rtcur(x, cfg)
        torch.cuda.synchronize()
        dt = 1e3 * (time.perf_counter() - t1)
        per.append(round(dt, 2))
        if dt > 12.0:   # a slow solve: where did the host time go
            tl = S._TIMELINE
            setup = [(tl[i][0], round(1e6 * (tl[i][2] - tl[i - 1][2]))) for i in range(1, len(tl)) if tl[i][1] == 0]
            print("  setup steps (us):", setup, flush=True)
            gaps = [(tl[i][0], tl[i][1], round(1e6 * (tl[i][2] - tl[i - 1][2]))) for i in range(1, len(tl))]
            print("  slow solve, largest host gaps (event, iteration, us since previous):",
                  sorted(gaps, key=lambda g: -g[2])[:6], " first event at",
                  round(1e6 * (tl[0][2] - t1)), "us", flush=True)
        S._TIMELINE = None
    torch.cuda.synchronize()
    print(f"{label:10s} {1e3 * (time.perf_counter() - t0) / 3:.2f} ms/solve  iters {res.iterations} "
          f"engines created {E.CREATED[0] - c0}  per solve {per}", flush=True)
S.PROFILE = False
