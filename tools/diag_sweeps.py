import json, math, sys, traceback
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200 import sweeps as sw
from paper_2108_10448_b200.synth import InstanceSpec, make_instance_device
from paper_2108_10448_b200.solver import SolverConfig, rtcur
from paper_2108_10448_b200.full import full_output
g = json.load(open("tests/golden/sweeps.json"))
a = g["phase_r"]["args"]
def trial(ia, iu, t):
    def run():
        alpha, upsilon = a["alphas"][ia], a["upsilons"][iu]
        inst_seed, solver_seed = sw._trial_seeds(0, ia, iu, t)
        spec = InstanceSpec(n=a["n"], d=a["d"], r=a["r"], alpha=alpha, seed=inst_seed)
        x, low, _ = make_instance_device(spec)
        try:
            cfg = SolverConfig(ranks=spec.ranks, eps=1e-5, zeta0=sw._inf_norm_dev(low), gamma=0.7, upsilon=upsilon,
                               variant="R", max_iters=a["max_iters"], seed=solver_seed)
            res = rtcur(x, cfg)
            est, _, _ = full_output(res, want_S=False)
            rel = float(torch.linalg.vector_norm(low.flat - est.flat.double()) / torch.linalg.vector_norm(low.flat))
            return ("ok", res.iterations, rel, res.error_history[-1])
        except Exception as ex:
            return ("EXC", repr(ex)[:200])
    return run
cells = [(0, iu, t) for iu in range(2) for t in range(3)]
ref = sw._run_parallel([trial(*c) for c in cells], 1)
print("ref", ref)
for rep in range(int(sys.argv[1])):
    for junk in (12345.678, -1e300, math.nan, 0.0):
        j = torch.full((96 * 1024 * 1024,), junk, dtype=torch.float64, device="cuda"); del j
        got = sw._run_parallel([trial(*c) for c in cells], 4)
        for c, r0, r1 in zip(cells, ref, got):
            if r0 != r1:
                print("DIFF rep", rep, "junk", junk, c, r0, "->", r1, flush=True)
print("done")
