"""Generate tests/golden/synth_instances.npz from the REAL reference's generator
(synth.py:74-135: gen_lowrank, gen_outliers, make_instance) for a few specs
covering both sampler branches (iid stream + first-unique, and permutation when
3k >= size), alpha = 0, n = 1 and n = 4.  Build container only.

Usage:  python tests/golden/make_synth_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402

SPECS = [(3, 12, 2, 0.2, 5), (2, 30, 3, 0.35, 7), (4, 6, 2, 0.05, 9), (1, 50, 1, 0.1, 3), (3, 12, 2, 0.0, 1),
         (3, 20, 3, 0.3, 11)]


def main():
    _import_reference()
    from rtcur.synth import InstanceSpec, make_instance

    out = {"specs": np.array(SPECS, dtype=np.float64)}
    for i, (n, d, r, a, s) in enumerate(SPECS):
        x, low, sparse = make_instance(InstanceSpec(n, d, r, a, s))
        out[f"x{i}"] = x.data
        out[f"low{i}"] = low.data
        out[f"sparse{i}"] = sparse.data
    np.savez_compressed(os.path.join(HERE, "synth_instances.npz"), **out)
    print("wrote synth_instances.npz", len(SPECS), "instances")


if __name__ == "__main__":
    main()
