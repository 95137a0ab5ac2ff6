"""Generate tests/golden/ap_hosvd.npz from the REAL reference's dense HOSVD
alternating-projections baseline (reference.py:132-193) on instances made by
its own make_instance (synth.py:124-135).  Build container only.

Usage:  python tests/golden/make_ap_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402

# (n, d, r, alpha, seed, use_true_zeta0, max_iters)
CASES = [(3, 16, 2, 0.1, 4, True, 60), (2, 40, 3, 0.2, 8, True, 80), (4, 8, 2, 0.05, 2, False, 60),
         (3, 12, 3, 0.0, 5, True, 40)]


def main():
    _import_reference()
    from rtcur.reference import ap_hosvd_trpca
    from rtcur.synth import InstanceSpec, make_instance
    from rtcur.tensor import inf_norm

    out = {"cases": np.array([[c[0], c[1], c[2], c[3], c[4], float(c[5]), c[6]] for c in CASES])}
    for i, (n, d, r, a, s, tz, mi) in enumerate(CASES):
        x, low, _ = make_instance(InstanceSpec(n, d, r, a, s))
        zeta0 = inf_norm(low) if tz else None
        L, S, hist = ap_hosvd_trpca(x, (r,) * n, zeta0=zeta0, gamma=0.7, eps=1e-5, max_iters=mi)
        out[f"x{i}"] = x.data
        out[f"zeta0_{i}"] = np.nan if zeta0 is None else zeta0
        out[f"L{i}"] = L.data
        out[f"S{i}"] = S.data
        out[f"hist{i}"] = np.array(hist)
    np.savez_compressed(os.path.join(HERE, "ap_hosvd.npz"), **out)
    print("wrote ap_hosvd.npz", len(CASES), "cases", [len(out[f"hist{i}"]) for i in range(len(CASES))])


if __name__ == "__main__":
    main()
