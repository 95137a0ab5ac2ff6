import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def solve_cases():
    return sorted(os.path.basename(p)[6:-4] for p in glob.glob(os.path.join(GOLDEN, "solve_*.npz")))


@pytest.fixture(scope="session")
def kernels_golden():
    return load_golden("kernels.npz")


def golden_cfg_kwargs(g):
    """SolverConfig keyword arguments recorded in a solve_*.npz fixture."""
    zeta0 = float(g["zeta0"])
    kw = dict(ranks=tuple(int(r) for r in g["ranks"]), eps=float(g["eps"]),
              zeta0=None if np.isnan(zeta0) else zeta0, gamma=float(g["gamma"]),
              upsilon=float(g["upsilon"]), variant=str(g["variant"]), max_iters=int(g["max_iters"]),
              seed=None if int(g["seed"]) < 0 else int(g["seed"]))
    if "row_sample_sizes" in g:
        kw["row_sample_sizes"] = tuple(int(v) for v in g["row_sample_sizes"])
    if "col_sample_sizes" in g:
        kw["col_sample_sizes"] = tuple(int(v) for v in g["col_sample_sizes"])
    return kw
