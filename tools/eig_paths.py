"""Diagnostic: which eigensolver path (warm subspace vs full) each mode takes per iteration, with the
clock64 marks of k_eig (full path: load, tridiagonalise, multisection, inverse iteration, back-transform;
warm path: load, setup + step 0, then step 1 split into K X, H + residual, certification, orthonormalisation)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200 import solver as S, synth
from paper_2108_10448_b200.fiber_cur import draw_sample_indices
from paper_2108_10448_b200.engine import acquire_engine
from paper_2108_10448_b200.tensor import DeviceTensor
from paper_2108_10448_b200 import _native as nat

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 3
if cfgi <= 1:
    x, _, _, bc = synth.make_config(cfgi)
    X = DeviceTensor(torch.from_numpy(x).cuda(), bc.shape)
else:
    X, bc = synth.make_config_device(cfgi)
rows, cols = synth.baseline_sample_sizes(bc.shape, bc.ranks)
cfg = S.SolverConfig(ranks=bc.ranks, variant=bc.variant, eps=bc.eps, gamma=0.7, seed=bc.seed_solver + 1000,
                     row_sample_sizes=rows, col_sample_sizes=cols)
lib = nat.load()
lib.rtcur_engine_debug_marks.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
src = S._Source(X)
rng = np.random.default_rng(cfg.seed)
rs, cs = cfg.resolve_sample_sizes(bc.shape)
print("rows", rs, "cols", cs, "ranks", bc.ranks)
idx = draw_sample_indices(bc.shape, rs, cs, rng)
eng = acquire_engine(bc.shape, bc.ranks, rs, cs, src.torch_dtype, slab=src.slab)
src.attach(eng); eng.set_sample(idx); src.load_blocks(eng, idx)
zeta = src.inf_norm(eng)
n = len(bc.shape)
buf = (ctypes.c_int64 * (9 * 8))()
clk = 1.92e3  # MHz approx for cycle->us
for k in range(1, 40):
    if cfg.variant == "R" and k >= 2:
        idx = draw_sample_indices(bc.shape, rs, cs, rng)
        eng.set_sample(idx); src.load_blocks(eng, idx)
    zeta *= cfg.gamma
    eng.iterate_async(zeta, first=(k == 1))
    e2, x2, fl = eng.iterate_wait()
    err = S._error_from_sums(e2, x2)
    lib.rtcur_engine_debug_marks(eng.handle, buf, 9 * 8)
    marks = np.frombuffer(buf, dtype=np.int64)
    m8 = marks[:8 * 8].reshape(8, 8)[:n]
    fast = marks[8 * 8:8 * 8 + n]
    span = [[round(int(r[j + 1] - r[j]) / clk, 2) if r[j+1] > 0 and r[j] > 0 else 0 for j in range(7)] for r in m8]
    # fast: > 0 warm-path steps, < 0 Lanczos steps (full path without Householder), 0 Householder
    print(f"it {k:2d} err {err:.3e} fast {[int(f) for f in fast]} eig_us {span}")
    if err <= cfg.eps:
        break
