"""Generate tests/golden/*.npz from the REAL reference (build container only).

Usage:  python tests/golden/make_golden.py
It builds (or reuses) a scratch copy of /root/reference/pkg with the Cython
backend (build_ref_scratch.sh), imports ``rtcur`` from it with
RTCUR_BACKEND=compiled, and records inputs + outputs of the reference's own
public API for the hot path:

* kernels.npz   sample_sizes / draw_sample_indices known answers, hard
                threshold, gather_columns, truncated_svd battery (linalg tests)
* solve_<case>.npz  full rtcur() solves (F and R, 1/3/4 modes, tall and wide
                intersections, zero tensor, clean low-rank, non-convergence)
                with per-iteration traces, the final FiberCur pieces and the
                full-output step (cli.py:237-243)
* cfg0_summary.npz  BASELINE config 0 (100^3, RTCUR-F) solved by the reference
                on the X produced by paper_2108_10448_b200.synth: error
                history, support bits, sampled L values and norms

The GPU box never runs this script (no /root/reference there); the committed
npz files travel with the repo.
"""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def _import_reference():
    src = subprocess.check_output(["bash", os.path.join(HERE, "build_ref_scratch.sh")], text=True).strip()
    os.environ["RTCUR_BACKEND"] = "compiled"
    sys.path.insert(0, src)
    import rtcur  # noqa: E402

    assert rtcur._backend.backend_name == "compiled"
    return rtcur


def _lowrank(rng, shape, ranks):
    from rtcur.tensor import DenseTensor, mode_product

    t = DenseTensor(rng.standard_normal(int(np.prod(ranks))), ranks)
    for m, (d, r) in enumerate(zip(shape, ranks), start=1):
        t = mode_product(t, rng.standard_normal((d, r)), m)
    return t


def _corrupt(rng, clean, alpha):
    """Reference test helper pattern (test_solver.py:25-36)."""
    from rtcur.tensor import DenseTensor

    total = clean.size
    count = int(alpha * total)
    pos = rng.permutation(total)[:count]
    mu = float(np.mean(np.abs(clean.data)))
    vals = rng.uniform(-mu, mu, size=count)
    data = np.array(clean.data)
    data[pos] += vals
    return DenseTensor(data, clean.shape)


def kernels(rtcur):
    from rtcur.fiber_cur import draw_sample_indices, sample_sizes
    from rtcur.linalg import truncated_svd
    from rtcur._backend import gather_columns, hard_threshold

    out = {}
    size_cases = [((300, 300, 300), (3, 3, 3), 3.0), ((10, 10, 10), (3, 3, 3), 1000.0),
                  ((1, 8), (1, 2), 0.001), ((9, 9, 9), (3, 3, 3), 0.001), ((40, 30, 20), (2, 2, 2), 3.0),
                  ((240, 320, 3, 600), (10, 10, 3, 2), 3.0), ((220,) * 4, (4,) * 4, 3.0)]
    for i, (shape, ranks, ups) in enumerate(size_cases):
        rows, cols = sample_sizes(shape, ranks, ups)
        out[f"sizes{i}_shape"] = np.array(shape)
        out[f"sizes{i}_ranks"] = np.array(ranks)
        out[f"sizes{i}_ups"] = np.array(ups)
        out[f"sizes{i}_rows"] = np.array(rows)
        out[f"sizes{i}_cols"] = np.array(cols)
    draw_cases = [((40, 30, 20), (6, 5, 4), (30, 40, 50), 42), ((10, 10, 10), (3, 9, 10), (5, 80, 100), 0),
                  ((400, 400, 400), (90, 90, 90), (2693, 2693, 2693), 1),
                  ((100, 100, 100), (42, 42, 42), (573, 573, 573), 0),
                  ((240, 320, 3, 600), (165, 174, 3, 39), (9012, 9983, 33, 492), 3),
                  ((220,) * 4, (65,) * 4, (1397,) * 4, 4), ((7,), (3,), (1,), 9)]
    for i, (shape, rs, cs, seed) in enumerate(draw_cases):
        rng = np.random.default_rng(seed)
        idx = draw_sample_indices(shape, rs, cs, rng)
        out[f"draw{i}_shape"] = np.array(shape)
        out[f"draw{i}_rs"] = np.array(rs)
        out[f"draw{i}_cs"] = np.array(cs)
        out[f"draw{i}_seed"] = np.array(seed)
        out[f"draw{i}_nrows"] = np.array(len(idx.rows))
        for m, r in enumerate(idx.rows):
            out[f"draw{i}_rows{m}"] = r
        for m, c in enumerate(idx.cols):
            out[f"draw{i}_cols{m}"] = c
        # a second draw from the same stream (RTCUR-R resample order)
        idx2 = draw_sample_indices(shape, rs, cs, rng)
        for m, c in enumerate(idx2.cols):
            out[f"draw{i}_cols{m}_second"] = c
    rng = np.random.default_rng(77)
    for i in range(6):
        x = rng.standard_normal(int(rng.integers(1, 3000)))
        z = float(abs(rng.standard_normal()))
        out[f"ht{i}_x"] = x
        out[f"ht{i}_z"] = np.array(z)
        out[f"ht{i}_y"] = np.asarray(hard_threshold(x.copy(), z))
    x = np.array([1.0, -1.0, 1.0000001, 0.0, -2.5])
    out["ht_edge_x"] = x
    out["ht_edge_y"] = np.asarray(hard_threshold(x.copy(), 1.0))
    for i in range(5):
        size = int(rng.integers(50, 600))
        flat = rng.standard_normal(size)
        stride = int(rng.integers(1, 5))
        length = int(rng.integers(1, 9))
        bases = rng.integers(0, size - stride * (length - 1), size=int(rng.integers(1, 12)))
        out[f"gather{i}_flat"] = flat
        out[f"gather{i}_bases"] = bases.astype(np.int64)
        out[f"gather{i}_stride"] = np.array(stride)
        out[f"gather{i}_length"] = np.array(length)
        out[f"gather{i}_out"] = np.asarray(gather_columns(flat, bases.astype(np.int64), stride, length))
    battery = [(rng.standard_normal((6, 4)), 3), (rng.standard_normal((4, 6)), 2),
               (rng.standard_normal((12, 12)), 5), (rng.standard_normal((30, 7)), 7),
               (rng.standard_normal((8, 2)) @ rng.standard_normal((2, 9)), 4), (np.zeros((5, 4)), 2),
               (np.diag([3.0, 2.0, 1.0]), 2), (rng.standard_normal((50, 50)), 11),
               (rng.standard_normal((1, 9)), 1), (rng.standard_normal((9, 1)), 1),
               (rng.standard_normal((42, 573)), 3), (rng.standard_normal((90, 700)), 5),
               (rng.standard_normal((213, 400)) * np.logspace(0, -3, 400)[None, :], 10)]
    for i, (m, r) in enumerate(battery):
        f = truncated_svd(m, r)
        out[f"svd{i}_m"] = m
        out[f"svd{i}_r"] = np.array(r)
        out[f"svd{i}_s"] = f.singular_values
        out[f"svd{i}_rec"] = f.reconstruct()
        out[f"svd{i}_pinv"] = f.pinv()
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def _save_solve(name, x, cfg, res, rtcur, keep_trace="all", full_output=True):
    from rtcur.fiber_cur import cur_reconstruct_full

    out = {"x": x.data.copy(), "shape": np.array(x.shape), "ranks": np.array(cfg.ranks),
           "eps": np.array(cfg.eps), "zeta0": np.array(np.nan if cfg.zeta0 is None else cfg.zeta0),
           "gamma": np.array(cfg.gamma), "upsilon": np.array(cfg.upsilon), "variant": np.array(cfg.variant),
           "max_iters": np.array(cfg.max_iters), "seed": np.array(-1 if cfg.seed is None else cfg.seed),
           "error_history": np.array(res.error_history), "iterations": np.array(res.iterations),
           "converged": np.array(res.converged), "diagnostics": np.array(res.diagnostics, dtype=bool),
           "zeta_final": np.array(res.zeta_final)}
    if cfg.row_sample_sizes is not None:
        out["row_sample_sizes"] = np.array(cfg.row_sample_sizes)
    if cfg.col_sample_sizes is not None:
        out["col_sample_sizes"] = np.array(cfg.col_sample_sizes)
    n = len(x.shape)
    cur = res.cur
    out["cur_core"] = cur.core.data.copy()
    for m in range(n):
        out[f"cur_fib{m}"] = cur.fibers[m]
        out[f"cur_factor{m}"] = cur.factors[m]
        out[f"cur_sv{m}"] = cur.intersections[m].singular_values
        out[f"cur_rec{m}"] = cur.intersections[m].reconstruct()
        out[f"rows{m}"] = res.sparse.indices.rows[m]
        out[f"cols{m}"] = res.sparse.indices.cols[m]
        out[f"s_fib{m}"] = res.sparse.fibers[m]
    out["s_core"] = np.asarray(res.sparse.core).reshape(-1, order="F")
    if res.trace is not None:
        iters = range(len(res.trace))
        if keep_trace != "all":
            iters = sorted(set([0, 1, 2, len(res.trace) - 1]) & set(range(len(res.trace))))
        out["trace_iters"] = np.array(list(iters))
        for t in iters:
            tr = res.trace[t]
            out[f"t{t}_zeta"] = np.array(tr["zeta"])
            out[f"t{t}_s_core"] = np.asarray(tr["s_core"]).reshape(-1, order="F")
            out[f"t{t}_l_core"] = np.asarray(tr["l_core"]).reshape(-1, order="F")
            for m in range(n):
                out[f"t{t}_s_fib{m}"] = tr["s_fibers"][m]
                out[f"t{t}_l_fib{m}"] = tr["l_fibers"][m]
                out[f"t{t}_rows{m}"] = tr["indices"].rows[m]
                out[f"t{t}_cols{m}"] = tr["indices"].cols[m]
    if full_output:
        low = cur_reconstruct_full(cur)
        sp = rtcur.hard_threshold(x.data - low.data, res.zeta_final)
        out["full_L"] = low.data.copy()
        out["full_S"] = np.asarray(sp)
    np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **out)
    print(f"solve_{name}: iters={res.iterations} conv={res.converged} err={res.error_history[-1]:.3e}")


def solves(rtcur):
    from rtcur import DenseTensor, SolverConfig, inf_norm
    from rtcur.synth import InstanceSpec, make_instance

    # test_reference.py:177-214 instance, both variants
    x, low, _ = make_instance(InstanceSpec(n=3, d=10, r=2, alpha=0.1, seed=3))
    for v in ("F", "R"):
        cfg = SolverConfig(ranks=(2, 2, 2), zeta0=inf_norm(low), upsilon=2.0, seed=5, variant=v, max_iters=60)
        _save_solve(f"d10_{v}", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur)
    # acceptance criterion 3 instance (d=20, F)
    x, low, _ = make_instance(InstanceSpec(n=3, d=20, r=2, alpha=0.1, seed=31))
    cfg = SolverConfig(ranks=(2, 2, 2), zeta0=inf_norm(low), upsilon=3.0, variant="F", seed=17, max_iters=80)
    _save_solve("d20_F", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur, keep_trace="some")
    # 4 modes, non-cubic, RTCUR-R, zeta0 = max|X|
    rng = np.random.default_rng(40)
    t = _lowrank(rng, (8, 9, 7, 6), (2, 2, 2, 2))
    x = _corrupt(rng, t, 0.1)
    cfg = SolverConfig(ranks=(2, 2, 2, 2), upsilon=3.0, seed=2, variant="R", max_iters=60)
    _save_solve("n4_R", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur, keep_trace="some")
    # tall mode-1 intersection (|I_1| = 21 > |J_1| = 16), mixed ranks, F
    rng = np.random.default_rng(41)
    t = _lowrank(rng, (30, 4, 4), (2, 2, 2))
    x = _corrupt(rng, t, 0.08)
    cfg = SolverConfig(ranks=(2, 2, 2), upsilon=3.0, seed=3, variant="F", max_iters=60,
                       zeta0=float(np.max(np.abs(t.data))))
    _save_solve("tall_F", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur, keep_trace="some")
    # non-cubic, mixed ranks, R
    rng = np.random.default_rng(42)
    t = _lowrank(rng, (16, 12, 10), (3, 2, 2))
    x = _corrupt(rng, t, 0.1)
    cfg = SolverConfig(ranks=(3, 2, 2), upsilon=3.0, seed=4, variant="R", max_iters=60,
                       zeta0=float(np.max(np.abs(t.data))))
    _save_solve("mixed_R", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur, keep_trace="some")
    # zero tensor (test_solver.py:172-179)
    x = DenseTensor.zeros((12, 10, 8))
    cfg = SolverConfig(ranks=(2, 2, 2), seed=0)
    _save_solve("zero", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur)
    # clean low rank (test_solver.py:122-130)
    rng = np.random.default_rng(1)
    x = _lowrank(rng, (20, 20, 20), (2, 2, 2))
    cfg = SolverConfig(ranks=(2, 2, 2), upsilon=4.0, eps=1e-8, seed=7)
    _save_solve("clean", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur)
    # non-convergence (test_solver.py:201-208)
    rng = np.random.default_rng(6)
    t = _lowrank(rng, (20, 20, 20), (2, 2, 2))
    x = _corrupt(rng, t, 0.1)
    cfg = SolverConfig(ranks=(2, 2, 2), eps=1e-300, max_iters=4, zeta0=float(np.max(np.abs(t.data))), seed=7)
    _save_solve("nonconv", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur)
    # single-mode tensor
    rng = np.random.default_rng(15)
    x = DenseTensor(rng.standard_normal(9) + np.where(rng.random(9) < 0.2, 5.0, 0.0), (9,))
    cfg = SolverConfig(ranks=(1,), seed=3, max_iters=20, upsilon=1.0)
    _save_solve("n1", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur)
    # BASELINE generator, small: Bernoulli support, c=10, baseline sample sizes, R
    sys.path.insert(0, ROOT)
    from paper_2108_10448_b200.synth import baseline_sample_sizes, make_gaussian_tucker

    shape, ranks = (30, 30, 30), (3, 3, 3)
    xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=77)
    rows, cols = baseline_sample_sizes(shape, ranks)
    cfg = SolverConfig(ranks=ranks, seed=8, variant="R", max_iters=100, row_sample_sizes=rows,
                       col_sample_sizes=cols)
    x = DenseTensor(xf, shape)
    _save_solve("bern_R", x, cfg, rtcur.rtcur(x, cfg, record_trace=True), rtcur, keep_trace="some")


def cfg0_summary(rtcur):
    """BASELINE config 0 on the synth X: store a compact summary of the result."""
    sys.path.insert(0, ROOT)
    from rtcur import DenseTensor, SolverConfig

    from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config

    xf, low, _, bc = make_config(0)
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, gamma=0.7, variant=bc.variant, max_iters=100,
                       seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols)
    x = DenseTensor(xf, bc.shape)
    res = rtcur.rtcur(x, cfg)
    out = {"error_history": np.array(res.error_history), "iterations": np.array(res.iterations),
           "converged": np.array(res.converged), "zeta_final": np.array(res.zeta_final),
           "diagnostics": np.array(res.diagnostics, dtype=bool)}
    n = 3
    rng = np.random.default_rng(123)
    s_core = np.asarray(res.sparse.core).reshape(-1, order="F")
    out["s_core_bits"] = np.packbits(s_core != 0.0)
    out["s_core_n"] = np.array(s_core.size)
    out["clean_core_norm"] = np.array(np.linalg.norm(res.cur.core.data))
    pos = rng.integers(0, s_core.size, 500)
    out["s_core_pos"] = pos
    out["s_core_val"] = s_core[pos]
    for m in range(n):
        s = np.asarray(res.sparse.fibers[m]).reshape(-1, order="F")
        out[f"s_fib{m}_bits"] = np.packbits(s != 0.0)
        out[f"s_fib{m}_n"] = np.array(s.size)
        p = rng.integers(0, s.size, 500)
        out[f"s_fib{m}_pos"] = p
        out[f"s_fib{m}_val"] = s[p]
        out[f"sv{m}"] = res.cur.intersections[m].singular_values
        fac = res.cur.factors[m]
        out[f"factor{m}_norm"] = np.array(np.linalg.norm(fac))
        out[f"rows{m}"] = res.sparse.indices.rows[m]
        out[f"cols{m}"] = res.sparse.indices.cols[m]
        out[f"clean_fib{m}_norm"] = np.array(np.linalg.norm(res.cur.fibers[m]))
    # low-rank estimate at 2000 random full-tensor positions + relative recovery
    from rtcur.fiber_cur import cur_reconstruct_full

    lf = cur_reconstruct_full(res.cur).data
    p = rng.integers(0, lf.size, 2000)
    out["L_pos"] = p
    out["L_val"] = lf[p]
    out["rel_recovery"] = np.array(np.linalg.norm(lf - low) / np.linalg.norm(low))
    np.savez_compressed(os.path.join(HERE, "cfg0_summary.npz"), **out)
    print(f"cfg0: iters={res.iterations} conv={res.converged} err={res.error_history[-1]:.3e} "
          f"rel={out['rel_recovery']:.2e} total={res.timings['total']:.2f}s")


if __name__ == "__main__":
    ref = _import_reference()
    kernels(ref)
    solves(ref)
    cfg0_summary(ref)
