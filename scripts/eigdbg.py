# diagnostics: per-phase clock64 marks inside k_eig on config 1 (not a test)
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur, _native
from paper_2108_10448_b200 import solver as sm
from paper_2108_10448_b200.synth import make_config, baseline_sample_sizes
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
xf, _, _, bc = make_config(cfgi)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
dt = torch.float64 if bc.dtype == "f64" else torch.float32
x = DeviceTensor(torch.from_numpy(xf).to(dt).cuda(), bc.shape)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=4, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
res = rtcur(x, cfg)
eng = res.cur._engine
lib = _native.load()
lib.rtcur_engine_debug_marks.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
buf = (ctypes.c_int64 * 64)()
_native.check(lib.rtcur_engine_debug_marks(eng.handle, buf, 64))
m = np.array(buf[:8 * len(bc.shape)]).reshape(len(bc.shape), 8)
names = ["load", "tridiag", "bisect", "inviter", "backtf"]
for k in range(len(bc.shape)):
    d = np.diff(m[k, :6])
    print("mode", k, " ".join(f"{n}={v/1.965e3:.1f}us" for n, v in zip(names, d)), f"total={(m[k,5]-m[k,0])/1.965e3:.1f}us")
