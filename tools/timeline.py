"""Diagnostic: per-phase device timeline of one profiled solve (all phases bracketed by events,
RTCUR_PROF_TIMELINE=1 prints every interval's start relative to the first iteration).
usage: RTCUR_PROF_TIMELINE=1 python tools/timeline.py <config> [first_seq last_seq] 2> tl.txt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200 import _native as nat  # noqa: E402
from paper_2108_10448_b200 import solver as S  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config, make_config_device  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if c <= 1:
    xf, _, _, bc = make_config(c)
    x = DeviceTensor(torch.from_numpy(xf).cuda(), bc.shape)
else:
    x, bc = make_config_device(c)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
S.PROFILE, S.PROFILE_PHASES = True, None
for _ in range(2):
    res = rtcur(x, cfg)
    res = None
torch.cuda.synchronize()
print("PHASES", " ".join(f"{i}={n}" for i, n in enumerate(nat.PHASES)), file=sys.stderr)
print("BEGIN", file=sys.stderr)
res = rtcur(x, cfg)
torch.cuda.synchronize()
