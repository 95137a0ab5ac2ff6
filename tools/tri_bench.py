"""Drive tools/tri_bench.cu: time the tridiagonalisation designs and check T's
eigenvalues against numpy.  python tools/tri_bench.py"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "_tri_bench.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(HERE, "tri_bench.cu")])
lib = ctypes.CDLL(so)
lib.tri_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
rng = np.random.default_rng(0)
for s in (42, 65, 90, 128):
    B = rng.standard_normal((s, 3 * s))
    K = B @ B.T
    ref = np.linalg.eigvalsh(K)
    Kd = torch.from_numpy(K.copy()).cuda()
    for variant in (0, 1):
        d = torch.zeros(s, dtype=torch.float64, device="cuda")
        e = torch.zeros(s, dtype=torch.float64, device="cuda")
        cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
        best = None
        for rep in range(5):
            st = lib.tri_run(Kd.data_ptr(), s, variant, d.data_ptr(), e.data_ptr(), cyc.data_ptr())
            assert st == 0, st
            c = int(cyc.item())
            best = c if best is None else min(best, c)
        T = np.diag(d.cpu().numpy()) + np.diag(e.cpu().numpy()[:s - 1], 1) + np.diag(e.cpu().numpy()[:s - 1], -1)
        ev = np.linalg.eigvalsh(T)
        err = float(np.max(np.abs(ev - ref)) / ref[-1])
        print(f"s={s:4d} variant={variant} {best / 1965.0:8.1f} us  ({best / (s - 2):.0f} cyc/step)  eig err {err:.1e}",
              flush=True)
