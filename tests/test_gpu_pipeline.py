"""The iteration pipeline (speculative launches with the device-side stop rule,
held-back tails, shadow iterates, side-stream staging, pooled-engine resets;
DESIGN.md §4.6) against the one-at-a-time loop the reference runs
(/root/reference/pkg/src/rtcur/solver.py:314-375: every iteration finished and
checked before the next starts): identical results on random small problems,
and run-to-run determinism at a BASELINE config."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, env.get("PYTHONPATH", "")])
    return subprocess.run([sys.executable] + args, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)


@pytest.mark.parametrize("seed", [3, 11])
def test_pipelined_loop_equals_one_at_a_time_on_random_problems(seed):
    r = _run([os.path.join(ROOT, "tools", "stress_pipeline.py"), "120", str(seed)])
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    assert " 0 mismatches" in r.stdout


def test_pipelined_solves_are_deterministic_run_to_run():
    r = _run([os.path.join(ROOT, "tools", "determinism.py"), "0", "12"])
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    assert "1 distinct result" in r.stdout
