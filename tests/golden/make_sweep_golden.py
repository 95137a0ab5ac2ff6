"""Generate tests/golden/sweeps.json from the REAL reference's sweep drivers
(synth.py:159-336): a small phase-transition grid (success counts) and a small
timing sweep (iteration counts; wall times are not comparable).  Build
container only.

Usage:  python tests/golden/make_sweep_golden.py
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402

PHASE = dict(alphas=(0.1, 0.3, 0.5), upsilons=(1.0, 3.0), trials=3, n=3, d=20, r=2, variant="F", max_iters=100)
PHASE_R = dict(alphas=(0.2,), upsilons=(2.0, 4.0), trials=3, n=3, d=16, r=2, variant="R", max_iters=100)
TIMING = dict(dims=(12, 18), methods=("rtcur-f", "rtcur-r", "hosvd-ap"), repeats=2, n=3, r=2, alpha=0.1,
              max_iters=200)


def main():
    _import_reference()
    from rtcur.synth import run_phase_transition, run_timing

    out = {}
    g = run_phase_transition(**PHASE)
    out["phase"] = {"args": {k: list(v) if isinstance(v, tuple) else v for k, v in PHASE.items()},
                    "successes": [list(r) for r in g.successes]}
    g = run_phase_transition(**PHASE_R)
    out["phase_r"] = {"args": {k: list(v) if isinstance(v, tuple) else v for k, v in PHASE_R.items()},
                      "successes": [list(r) for r in g.successes]}
    rows = run_timing(**TIMING)
    out["timing"] = {"args": {k: list(v) if isinstance(v, tuple) else v for k, v in TIMING.items()},
                     "rows": [{"d": r.d, "method": r.method, "iters": r.iters, "censored": r.censored} for r in rows]}
    with open(os.path.join(HERE, "sweeps.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote sweeps.json", out["phase"]["successes"], out["phase_r"]["successes"],
          [(r["d"], r["method"], r["iters"]) for r in out["timing"]["rows"]])


if __name__ == "__main__":
    main()
