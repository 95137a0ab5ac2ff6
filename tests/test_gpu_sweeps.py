"""Batched sweeps on the GPU vs the real reference's drivers on
the same seeds (tests/golden/sweeps.json)."""

import json
import os

import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with open(os.path.join(GOLDEN, "sweeps.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("key", ["phase", "phase_r"])
@pytest.mark.parametrize("workers", [1, 4])
def test_phase_transition_matches_reference(golden, key, workers):
    from paper_2108_10448_b200.sweeps import run_phase_transition

    a = dict(golden[key]["args"])
    seen = []
    g = run_phase_transition(workers=workers, progress=lambda *t: seen.append(t), **a)
    assert [list(r) for r in g.successes] == golden[key]["successes"]
    assert len(seen) == len(a["alphas"]) * len(a["upsilons"]) * a["trials"]
    csv = g.to_csv().strip().split("\n")
    assert csv[0] == "alpha,upsilon,successes,trials" and len(csv) == 1 + len(a["alphas"]) * len(a["upsilons"])


def test_timing_iterations_match_reference(golden):
    from paper_2108_10448_b200.sweeps import run_timing, timing_to_csv

    a = dict(golden["timing"]["args"])
    rows = run_timing(**a)
    assert [(r.d, r.method) for r in rows] == [(x["d"], x["method"]) for x in golden["timing"]["rows"]]
    for r, x in zip(rows, golden["timing"]["rows"]):
        assert r.iters == x["iters"], (r.d, r.method)
        assert r.mean_s > 0 and not r.censored
    assert timing_to_csv(rows).startswith("d,method,mean_s,std_s,iters,censored\n")
