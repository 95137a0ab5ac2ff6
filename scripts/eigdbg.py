# diagnostics: per-iteration eigensolver path (fast subspace iteration vs full) and clock64 phase marks
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, _native
from paper_2108_10448_b200.engine import Engine
from paper_2108_10448_b200.fiber_cur import draw_sample_indices
from paper_2108_10448_b200.synth import make_config, baseline_sample_sizes
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 25
xf, _, _, bc = make_config(cfgi)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
dt = torch.float64 if bc.dtype == "f64" else torch.float32
x = DeviceTensor(torch.from_numpy(xf).to(dt).cuda(), bc.shape)
eng = Engine(bc.shape, bc.ranks, rows, cols, dt)
eng.bind(x.flat)
rng = np.random.default_rng(bc.seed_solver)
lib = _native.load()
lib.rtcur_engine_debug_marks.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
zeta = eng.absmax()
n = len(bc.shape)
for k in range(1, iters + 1):
    if k == 1 or bc.variant == "R":
        idx = draw_sample_indices(bc.shape, rows, cols, rng)
        eng.set_sample(idx)
        eng.gather()
    zeta *= 0.7
    e2, x2, fl = eng.iterate(zeta, first=(k == 1))
    err = float(np.sum(np.sqrt(e2)) / np.sum(np.sqrt(x2)))
    buf = (ctypes.c_int64 * 72)()
    _native.check(lib.rtcur_engine_debug_marks(eng.handle, buf, 72))
    m = np.array(buf[:64]).reshape(8, 8)[:n]
    fast = list(buf[64:64 + n])
    tot = [(m[j, 5] - m[j, 0]) / 1.965e3 for j in range(n)]
    print(f"iter {k:2d} err={err:.3e} fast={fast} eig_us={[round(t, 1) for t in tot]}")
