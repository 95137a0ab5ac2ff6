"""Diagnostic: where the end-to-end (host buffers in/out) time of one solve goes."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200 import solver as S, synth
from paper_2108_10448_b200.tensor import DeviceTensor

x, _, _, bc = synth.make_config(1)
rows, cols = synth.baseline_sample_sizes(bc.shape, bc.ranks)
cfg = S.SolverConfig(ranks=bc.ranks, variant=bc.variant, eps=bc.eps, gamma=0.7, seed=bc.seed_solver + 1000,
                     row_sample_sizes=rows, col_sample_sizes=cols)
pinned = torch.from_numpy(x).pin_memory()
buf = torch.empty(pinned.numel(), dtype=torch.float64, device="cuda")
for rep in range(4):
    t = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    buf.copy_(pinned, non_blocking=True); torch.cuda.synchronize(); t["h2d"] = time.perf_counter() - t0
    t0 = time.perf_counter(); res = S.rtcur(DeviceTensor(buf, bc.shape), cfg); t["solve"] = time.perf_counter() - t0
    t0 = time.perf_counter(); sc = res.sparse.core; t["sparse.core(+blocks)"] = time.perf_counter() - t0
    t0 = time.perf_counter(); sf = res.sparse.fibers; t["sparse.fibers"] = time.perf_counter() - t0
    t0 = time.perf_counter(); core = res.cur.core; t["cur.core"] = time.perf_counter() - t0
    t0 = time.perf_counter(); fib = res.cur.fibers; t["cur.fibers"] = time.perf_counter() - t0
    t0 = time.perf_counter(); it = res.cur.intersections; t["intersections"] = time.perf_counter() - t0
    t0 = time.perf_counter(); fa = res.cur.factors; t["factors"] = time.perf_counter() - t0
    tot = sum(t.values())
    print(f"rep {rep}: total {tot*1e3:.1f} ms  " + "  ".join(f"{k} {v*1e3:.1f}" for k, v in t.items()))

# inside the export: device export kernel, D2H into the pinned stage, host copies
from paper_2108_10448_b200 import engine as E
orig = E.Engine.to_host


def timed_to_host(self, dev):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    total = sum(int(t.numel()) for t in dev)
    st = getattr(self, "_pin_stage", None)
    if st is None or st.numel() < total:
        st = self._pin_stage = torch.empty(total, dtype=torch.float64, pin_memory=True)
    o = 0
    for t in dev:
        st[o:o + t.numel()].copy_(t, non_blocking=True)
        o += t.numel()
    torch.cuda.current_stream(self.device).synchronize()
    t1 = time.perf_counter()
    out = orig(self, dev)
    t2 = time.perf_counter()
    print(f"    to_host {total * 8 / 1e6:.1f} MB: d2h {1e3 * (t1 - t0):.2f} ms, full to_host {1e3 * (t2 - t1):.2f} ms")
    return out


E.Engine.to_host = timed_to_host
orig_eb = E.Engine.export_blocks


def timed_eb(self, *a):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = orig_eb(self, *a)
    torch.cuda.synchronize()
    print(f"    export_blocks (device) {1e3 * (time.perf_counter() - t0):.2f} ms")
    return out


E.Engine.export_blocks = timed_eb
for rep in range(2):
    res = None
    buf.copy_(pinned, non_blocking=True)
    res = S.rtcur(DeviceTensor(buf, bc.shape), cfg)
    t0 = time.perf_counter()
    _ = (res.sparse.core, res.sparse.fibers, res.cur.core, res.cur.fibers, res.cur.intersections, res.cur.factors)
    print(f"  export total {1e3 * (time.perf_counter() - t0):.2f} ms")
