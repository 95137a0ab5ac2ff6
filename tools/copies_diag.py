"""Diagnostic: where the per-solve mode-copy setup time goes (mem_get_info / allocation / transposes)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur  # noqa: E402
from paper_2108_10448_b200 import engine as E  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config  # noqa: E402

xf, _, _, bc = make_config(1)
x = DeviceTensor(torch.from_numpy(xf).cuda(), bc.shape)
rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                   row_sample_sizes=rows, col_sample_sizes=cols)
orig_bind = E.Engine.bind_mode_copies
orig_mgi = torch.cuda.mem_get_info
orig_empty_like = torch.empty_like
T = {}


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


E.Engine.bind_mode_copies = timed("bind_mode_copies", orig_bind)
torch.cuda.mem_get_info = timed("mem_get_info", orig_mgi)
torch.empty_like = timed("empty_like", orig_empty_like)
import ctypes  # noqa: E402
from paper_2108_10448_b200 import _native as nat  # noqa: E402
lib = nat.load()
for nm in ("rtcur_transpose_mode", "rtcur_engine_bind", "rtcur_engine_profile", "rtcur_engine_profile_read"):
    pass
orig_attach = S_attach = None
from paper_2108_10448_b200 import solver as S  # noqa: E402
S._Source.attach = timed("attach", S._Source.attach)
S._mode_copy_plan = timed("mode_copy_plan", S._mode_copy_plan)
S.acquire_engine = timed("acquire_engine", S.acquire_engine)
for i in range(80):
    T.clear()
    res = None
    t0 = time.perf_counter()
    res = rtcur(x, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = torch.cuda.memory_stats()
    if dt > 0.010:
      print(f"solve {i}: {1e3 * dt:.2f} ms  " + "  ".join(f"{k} {1e3 * v:.2f}" for k, v in T.items())
          + f"  reserved {st['reserved_bytes.all.current'] >> 20} MB, cudaMalloc calls {st['num_device_alloc']}, frees {st['num_device_free']}")
