"""Uninitialised-memory / race hunt on the batched sweeps: poison the caching
allocator with different junk before each phase-transition run (4 workers) and
compare the per-trial outcomes with the golden counts.

usage: python tools/poison_sweeps.py [key] [reps]
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200.sweeps import run_phase_transition  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "phase_r"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "sweeps.json")))
a = dict(g[key]["args"])
want = g[key]["successes"]
bad = 0
for rep in range(reps):
    for junk in (12345.678, -1e300, math.nan, 0.0):
        j = torch.full((96 * 1024 * 1024,), junk, dtype=torch.float64, device="cuda")
        del j
        for w in (1, 4):
            got = [list(r) for r in run_phase_transition(workers=w, **a).successes]
            if got != want:
                bad += 1
                print("MISMATCH rep", rep, "junk", junk, "workers", w, got, "want", want, flush=True)
print("done", key, "mismatches", bad)
