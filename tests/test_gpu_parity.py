"""GPU parity: the sm_100a path (through librtcur_b200.so) against the
reference's golden vectors and the CPU oracle on identical inputs and
identical sampled index sets.

Bars (north_star + reference tests): index sets bit-exact; recovered sparse
support bit-exact; S/L blocks and errors within 1e-10 absolute in fp64
(test_reference.py:177-214); iteration counts and convergence identical;
singular values 1e-10 relative; full-output L/S 1e-8 (test_reference.py:217).
fp32 inputs: compared against the fp64 oracle run on the exactly-upcast X,
tolerance 1e-4 relative Frobenius (BASELINE north_star), support bit-exact.
"""

import numpy as np
import pytest

from conftest import golden_cfg_kwargs, load_golden, solve_cases

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, run on the B200
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import rtcur_oracle as orc  # noqa: E402
from paper_2108_10448_b200 import (DenseTensor, DeviceTensor, SolverConfig, cur_reconstruct_full,  # noqa: E402
                                   full_output, hard_threshold, rtcur)
from paper_2108_10448_b200 import _native  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config, make_gaussian_tucker  # noqa: E402


def _flat(a):
    return np.asarray(a).reshape(-1, order="F")


@pytest.mark.parametrize("case", solve_cases())
def test_solve_matches_reference_golden(case):
    g = load_golden(f"solve_{case}.npz")
    shape = tuple(int(d) for d in g["shape"])
    n = len(shape)
    cfg = SolverConfig(**golden_cfg_kwargs(g))
    res = rtcur(DenseTensor(g["x"], shape), cfg, record_trace=True)
    assert res.iterations == int(g["iterations"])
    assert res.converged == bool(g["converged"])
    np.testing.assert_allclose(res.error_history, g["error_history"], atol=1e-10, rtol=0)
    assert np.array_equal(np.array(res.diagnostics, dtype=bool).reshape(g["diagnostics"].shape), g["diagnostics"])
    assert res.zeta_final == pytest.approx(float(g["zeta_final"]), rel=1e-15)
    for t in g["trace_iters"]:
        tr = res.trace[int(t)]
        for m in range(n):
            assert np.array_equal(tr["indices"].rows[m], g[f"t{t}_rows{m}"])
            assert np.array_equal(tr["indices"].cols[m], g[f"t{t}_cols{m}"])
        for key in ("s_core", "l_core"):
            got, want = _flat(tr[key]), g[f"t{t}_{key}"]
            np.testing.assert_allclose(got, want, atol=1e-10, rtol=0, err_msg=f"iter {t} {key}")
        assert np.array_equal(_flat(tr["s_core"]) != 0, g[f"t{t}_s_core"] != 0)
        for m in range(n):
            np.testing.assert_allclose(tr["s_fibers"][m], g[f"t{t}_s_fib{m}"], atol=1e-10, rtol=0)
            np.testing.assert_allclose(tr["l_fibers"][m], g[f"t{t}_l_fib{m}"], atol=1e-10, rtol=0)
            assert np.array_equal(tr["s_fibers"][m] != 0, g[f"t{t}_s_fib{m}"] != 0)
    # final SolveResult pieces
    np.testing.assert_allclose(_flat(res.sparse.core), g["s_core"], atol=1e-10, rtol=0)
    assert np.array_equal(_flat(res.sparse.core) != 0, g["s_core"] != 0)
    np.testing.assert_allclose(res.cur.core.data, g["cur_core"], atol=1e-10, rtol=0)
    for m in range(n):
        assert np.array_equal(res.sparse.indices.cols[m], g[f"cols{m}"])
        np.testing.assert_allclose(res.sparse.fibers[m], g[f"s_fib{m}"], atol=1e-10, rtol=0)
        np.testing.assert_allclose(res.cur.fibers[m], g[f"cur_fib{m}"], atol=1e-10, rtol=0)
        sv = res.cur.intersections[m].singular_values
        scale = max(1.0, float(g[f"cur_sv{m}"][0]))
        np.testing.assert_allclose(sv, g[f"cur_sv{m}"], atol=1e-10 * scale, rtol=0)
        np.testing.assert_allclose(res.cur.intersections[m].reconstruct(), g[f"cur_rec{m}"], atol=1e-9 * scale)
        np.testing.assert_allclose(res.cur.factors[m], g[f"cur_factor{m}"], atol=1e-8)
    # full-output step (cli.py:237-243)
    L, S, _ = full_output(res)
    np.testing.assert_allclose(L.flat.cpu().numpy(), g["full_L"], atol=1e-8)
    np.testing.assert_allclose(S.flat.cpu().numpy(), g["full_S"], atol=1e-8)
    np.testing.assert_allclose(cur_reconstruct_full(res.cur).data, g["full_L"], atol=1e-8)


def test_cfg0_matches_reference_summary():
    g = load_golden("cfg0_summary.npz")
    xf, _, _, bc = make_config(0)
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100, seed=bc.seed_solver,
                       row_sample_sizes=rows, col_sample_sizes=cols)
    res = rtcur(DeviceTensor.from_host(xf.reshape(bc.shape, order="F")), cfg)
    assert res.iterations == int(g["iterations"])
    np.testing.assert_allclose(res.error_history, g["error_history"], atol=1e-10, rtol=0)
    s_core = _flat(res.sparse.core)
    assert np.array_equal(np.packbits(s_core != 0), g["s_core_bits"])
    np.testing.assert_allclose(s_core[g["s_core_pos"]], g["s_core_val"], atol=1e-10)
    for m in range(3):
        s = _flat(res.sparse.fibers[m])
        assert np.array_equal(np.packbits(s != 0), g[f"s_fib{m}_bits"])
        np.testing.assert_allclose(s[g[f"s_fib{m}_pos"]], g[f"s_fib{m}_val"], atol=1e-10)
        np.testing.assert_allclose(res.cur.intersections[m].singular_values, g[f"sv{m}"], rtol=1e-10)
        assert np.array_equal(res.sparse.indices.cols[m], g[f"cols{m}"])
    L, _, _ = full_output(res, want_S=False)
    np.testing.assert_allclose(L.flat.cpu().numpy()[g["L_pos"]], g["L_val"], atol=1e-9)


@pytest.mark.parametrize("variant", ["F", "R"])
def test_fp32_storage_matches_fp64_oracle(variant):
    """fp32-stored X (configs 2-4 precision): GPU computes in fp64 on the exact
    upcast, so it must track the fp64 oracle run on the same values."""
    shape, ranks = (40, 36, 30), (3, 3, 3)
    xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=21, dtype=np.float32)
    rows, cols = baseline_sample_sizes(shape, ranks)
    kw = dict(eps=1e-5, variant=variant, max_iters=100, seed=4, row_sample_sizes=rows, col_sample_sizes=cols)
    dev = DeviceTensor(torch.from_numpy(xf).cuda(), shape)
    res = rtcur(dev, SolverConfig(ranks=ranks, **kw))
    ref = orc.solve(xf.astype(np.float64), shape, ranks, **kw)
    assert res.iterations == ref.iterations and res.converged == ref.converged
    np.testing.assert_allclose(res.error_history, ref.error_history, atol=1e-10, rtol=0)
    s_core = _flat(res.sparse.core)
    r_core = _flat(ref.s_core)
    assert np.array_equal(s_core != 0, r_core != 0)
    assert np.linalg.norm(s_core - r_core) <= 1e-4 * max(np.linalg.norm(r_core), 1e-300)
    for m in range(3):
        assert np.array_equal(res.sparse.fibers[m] != 0, ref.s_fibers[m] != 0)
        rel = np.linalg.norm(res.sparse.fibers[m] - ref.s_fibers[m]) / max(np.linalg.norm(ref.s_fibers[m]), 1e-300)
        assert rel <= 1e-4
    low, sp, e2, x2 = orc.full_output(xf.astype(np.float64), shape, ref.cur, ref.zeta_final)
    L, S, rel = full_output(res)
    Lh = L.flat.double().cpu().numpy()
    assert np.linalg.norm(Lh - low) <= 1e-4 * np.linalg.norm(low)
    assert rel == pytest.approx(np.sqrt(e2 / x2), rel=1e-3, abs=1e-7)


def test_kernel_plug_hard_threshold_and_gather(kernels_golden):
    g = kernels_golden
    for i in range(6):
        y = hard_threshold(g[f"ht{i}_x"], float(g[f"ht{i}_z"]))
        assert np.array_equal(y, g[f"ht{i}_y"])
    assert np.array_equal(hard_threshold(g["ht_edge_x"], 1.0), g["ht_edge_y"])
    with pytest.raises(ValueError):
        hard_threshold(np.ones(3), -0.1)
    lib = _native.load()
    st = torch.cuda.current_stream().cuda_stream
    for i in range(5):
        flat = torch.from_numpy(g[f"gather{i}_flat"]).cuda()
        bases = torch.from_numpy(g[f"gather{i}_bases"]).cuda()
        stride, length = int(g[f"gather{i}_stride"]), int(g[f"gather{i}_length"])
        out = torch.empty(length * bases.numel(), dtype=torch.float64, device="cuda")
        _native.check(lib.rtcur_gather_columns(flat.data_ptr(), 0, flat.numel(), bases.data_ptr(), bases.numel(),
                                               stride, length, out.data_ptr(), st))
        got = out.cpu().numpy().reshape((length, bases.numel()), order="F")
        assert np.array_equal(got, g[f"gather{i}_out"])
    bad = torch.tensor([5], dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        _native.check(lib.rtcur_gather_columns(flat.data_ptr(), 0, 6, bad.data_ptr(), 1, 1, 3, out.data_ptr(), st))


def test_kernel_plug_truncated_svd_battery(kernels_golden):
    g = kernels_golden
    lib = _native.load()
    st = torch.cuda.current_stream().cuda_stream
    i = 0
    while f"svd{i}_m" in g:
        m, r = g[f"svd{i}_m"], int(g[f"svd{i}_r"])
        a = torch.from_numpy(np.asfortranarray(m).reshape(-1, order="F").copy()).cuda()
        u = torch.empty(m.shape[0] * r, dtype=torch.float64, device="cuda")
        v = torch.empty(m.shape[1] * r, dtype=torch.float64, device="cuda")
        s = torch.empty(r, dtype=torch.float64, device="cuda")
        _native.check(lib.rtcur_truncated_svd(a.data_ptr(), m.shape[0], m.shape[1], r, u.data_ptr(), s.data_ptr(),
                                              v.data_ptr(), st))
        U = u.cpu().numpy().reshape((m.shape[0], r), order="F")
        V = v.cpu().numpy().reshape((m.shape[1], r), order="F")
        S = s.cpu().numpy()
        scale = max(float(g[f"svd{i}_s"][0]), 1.0)
        np.testing.assert_allclose(S, g[f"svd{i}_s"], atol=1e-10 * scale, err_msg=f"case {i}")
        np.testing.assert_allclose((U * S) @ V.T, g[f"svd{i}_rec"], atol=1e-9 * scale, err_msg=f"case {i}")
        np.testing.assert_allclose(U.T @ U, np.eye(r), atol=1e-10, err_msg=f"case {i}")
        np.testing.assert_allclose(V.T @ V, np.eye(r), atol=1e-10, err_msg=f"case {i}")
        i += 1


def test_errors_mirror_reference():
    t = DenseTensor.zeros((5, 5, 5))
    with pytest.raises(ValueError):
        rtcur(t, SolverConfig(ranks=(6, 2, 2)))
    with pytest.raises(ValueError):
        rtcur(t, SolverConfig(ranks=(2, 2)))
    x = np.zeros((6, 6, 6))
    x[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        rtcur(DenseTensor.from_array(x), SolverConfig(ranks=(2, 2, 2), seed=1, zeta0=1.0, upsilon=10.0))


def test_native_code_ran():
    assert _native.launch_count() > 0


@pytest.mark.gpu
def test_graph_captured_iterations_match():
    """Per-iteration CUDA graphs (the default; zeta from device memory) give the same
    iterates as the stream-launched path (RTCUR_GRAPHS=0), R and F, several slot rotations."""
    import os
    import subprocess
    import sys

    code = r'''
import sys
sys.path.insert(0, ".")
from conftest import load_golden, golden_cfg_kwargs
from paper_2108_10448_b200 import SolverConfig, rtcur
from paper_2108_10448_b200.tensor import DenseTensor
for case in ("bern_R", "d20_F", "n4_R"):
    g = load_golden(f"solve_{case}.npz")
    shape = tuple(int(v) for v in g["shape"])
    res = rtcur(DenseTensor(g["x"], shape), SolverConfig(**golden_cfg_kwargs(g)))
    print(case, res.iterations, repr(list(res.error_history)))
'''
    outs = []
    here = os.path.dirname(os.path.abspath(__file__))
    for env in ({"RTCUR_GRAPHS": "0"}, {"RTCUR_GRAPHS": "1"}):
        e = dict(os.environ, **env)
        e["PYTHONPATH"] = os.pathsep.join([os.path.dirname(here), here, e.get("PYTHONPATH", "")])
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, cwd=here)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout)
    assert outs[0] == outs[1] and outs[0].count("\n") == 3


@pytest.mark.parametrize("case", ["bern_R", "d20_F", "n4_R", "nonconv", "zero", "n1"])
def test_speculative_pipeline_matches_one_at_a_time(case):
    """The speculative loop (iteration k + 1 enqueued behind k, cancelled on the device
    when k meets the stop rule, solver.py:357-358) returns what the one-at-a-time loop
    returns: iterates, index sets, exported blocks, factors -- also when the solve stops
    at max_iters (no iteration enqueued past it) and when the next solve reuses the
    pooled engine after a cancel."""
    from paper_2108_10448_b200 import solver as S

    g = load_golden(f"solve_{case}.npz")
    shape = tuple(int(d) for d in g["shape"])
    kw = golden_cfg_kwargs(g)
    x = DeviceTensor.from_host(DenseTensor(g["x"], shape))
    full_iters = int(g["iterations"])
    for max_iters in (kw["max_iters"], 1, 2, max(1, full_iters - 1)):
        cfg = SolverConfig(**dict(kw, max_iters=max_iters))
        got = {}
        for spec in (False, True, True):   # (twice: the pooled engine right after a cancel)
            S.SPECULATE = spec
            try:
                res = rtcur(x, cfg)
                got[spec] = (res.iterations, res.converged, tuple(res.error_history), res.zeta_final,
                             [np.array(r) for r in res.sparse.indices.rows], [np.array(c) for c in res.sparse.indices.cols],
                             _flat(res.sparse.core).copy(), [np.array(f) for f in res.sparse.fibers],
                             _flat(res.cur.core.data).copy(), [np.array(t.singular_values) for t in res.cur.intersections],
                             [np.array(f) for f in res.cur.factors], tuple(res.diagnostics))
            finally:
                S.SPECULATE = True
            del res
        a, b = got[False], got[True]
        assert a[:4] == b[:4] and a[11] == b[11], (max_iters, a[:2], b[:2])
        for i in (4, 5, 7, 9, 10):
            assert len(a[i]) == len(b[i])
            for u, v in zip(a[i], b[i]):
                assert np.array_equal(u, v), (max_iters, i)
        assert np.array_equal(a[6], b[6]) and np.array_equal(a[8], b[8])


@pytest.mark.parametrize("env", [{"RTCUR_FIBER_PASS": "0"}, {"RTCUR_FIBER_CORE": "0"}, {"RTCUR_EARLY_ZETA": "0"},
                                 {"RTCUR_K3_GENERIC": "1"}, {"RTCUR_CORE_PASS": "1"}, {"RTCUR_EIG_REG": "0"},
                                 {"RTCUR_EIG_REG": "2"}, {"RTCUR_SIDE_PREFETCH": "0"}, {"RTCUR_SPECULATE": "0"},
                                 {"RTCUR_TAIL_DEFER": "0"}, {"RTCUR_TAIL_DEFER": "1"}, {"RTCUR_SHADOW": "0"},
                                 {"RTCUR_STAGE_LATE": "0"}, {"RTCUR_EIG_KFULL": "0"}, {"RTCUR_GRAPHS": "0"}],
                         ids=["block-pass-only", "core-on-block-pass", "late-zeta0", "generic-k3", "core-pass",
                              "eig-smem-tridiag", "eig-reg-tridiag", "in-order-prefetch", "one-at-a-time",
                              "tail-in-order", "tail-held-back", "no-shadow", "stage-under-eig", "packed-lanczos-matvec",
                              "no-graphs"])
def test_engine_variants_agree(env):
    """The device-path variants (TMA fiber pass vs the block pass for every block,
    the core on either, zeta_0 scanned before or after the first draw, TMA vs
    generic K3, and the pipeline's switches: speculation, held-back tail, shadow
    iterate, staging point, graphs) solve the golden cases identically: same iteration counts and
    sparse support; the error histories and the full-output residual to 1e-9
    relative (the A pass and the sums group their fixed-order additions
    differently, ~1e-16 of L, amplified by 1/e ~ 1e5 in the relative residuals)."""
    import os
    import subprocess
    import sys

    code = r'''
import sys
sys.path.insert(0, ".")
import numpy as np
from conftest import load_golden, golden_cfg_kwargs
from paper_2108_10448_b200 import SolverConfig, rtcur, full_output
from paper_2108_10448_b200.tensor import DenseTensor
for case in ("bern_R", "d20_F", "n4_R", "tall_F"):
    g = load_golden(f"solve_{case}.npz")
    shape = tuple(int(v) for v in g["shape"])
    res = rtcur(DenseTensor(g["x"], shape), SolverConfig(**golden_cfg_kwargs(g)))
    _, _, rel = full_output(res)
    supp = int(np.count_nonzero(res.sparse.core)) + sum(int(np.count_nonzero(f)) for f in res.sparse.fibers)
    print(case, res.iterations, supp, repr(rel), repr(list(res.error_history)))
'''
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for e_ in ({}, env):
        e = dict(os.environ, **e_)
        e["PYTHONPATH"] = os.pathsep.join([os.path.dirname(here), here, e.get("PYTHONPATH", "")])
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, cwd=here)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append([ln.split(" ", 4) for ln in r.stdout.strip().splitlines()])
    assert len(outs[0]) == len(outs[1]) == 4
    for a, b in zip(*outs):
        assert a[:3] == b[:3], (a[:3], b[:3])   # case, iterations, support size
        assert float(a[3]) == pytest.approx(float(b[3]), rel=1e-9, abs=1e-300)
        np.testing.assert_allclose(eval(a[4]), eval(b[4]), rtol=1e-9, atol=0)


def test_solve_on_recycled_device_memory():
    """Regression for reads of never-written workspace: fill the caching allocator's
    memory with junk first, then solve a fresh geometry whose blocks split between the
    fiber pass and the block pass (a mode-3 fiber block with 4-byte-misaligned columns)
    and compare with the fp64 oracle (iterations, error history, support)."""
    junk = torch.full((96 * 1024 * 1024,), 12345.678, dtype=torch.float64, device="cuda")
    del junk
    shape, ranks = (44, 36, 30), (3, 2, 3)
    xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=23, dtype=np.float32)
    rows, cols = baseline_sample_sizes(shape, ranks)
    kw = dict(eps=1e-5, variant="F", max_iters=100, seed=5, row_sample_sizes=rows, col_sample_sizes=cols)
    res = rtcur(DeviceTensor(torch.from_numpy(xf).cuda(), shape), SolverConfig(ranks=ranks, **kw))
    ref = orc.solve(xf.astype(np.float64), shape, ranks, **kw)
    assert res.iterations == ref.iterations and res.converged == ref.converged
    np.testing.assert_allclose(res.error_history, ref.error_history, atol=1e-10, rtol=0)
    assert np.array_equal(_flat(res.sparse.core) != 0, _flat(ref.s_core) != 0)
    for m in range(3):
        assert np.array_equal(res.sparse.fibers[m] != 0, ref.s_fibers[m] != 0)


def test_sparse_estimate_outlives_its_result():
    """res.sparse must keep its own blocks after the SolveResult is dropped and a
    same-geometry solve reuses the pooled engine (reference SparseEstimate holds
    arrays, solver.py:121-127)."""
    import gc

    shape, ranks = (24, 20, 16), (2, 2, 2)
    rows, cols = baseline_sample_sizes(shape, ranks)
    kw = dict(ranks=ranks, eps=1e-5, variant="F", max_iters=60, row_sample_sizes=rows, col_sample_sizes=cols)
    xa, _, _ = make_gaussian_tucker(shape, ranks, 0.15, 10.0, seed=5)
    xb, _, _ = make_gaussian_tucker(shape, ranks, 0.25, 10.0, seed=6)
    want = orc.solve(xa, shape, ranks, **{k: v for k, v in kw.items() if k != "ranks"}, seed=3)
    res = rtcur(DenseTensor(xa, shape), SolverConfig(seed=3, **kw))
    sp = res.sparse
    del res
    gc.collect()
    other = rtcur(DenseTensor(xb, shape), SolverConfig(seed=4, **kw))
    np.testing.assert_allclose(_flat(sp.core), _flat(want.s_core), atol=1e-10)
    for m in range(3):
        np.testing.assert_allclose(sp.fibers[m], want.s_fibers[m], atol=1e-10)
    assert other.iterations >= 1


def test_dense_accessor_methods_match_oracle():
    """DenseTensorAccessor.core_block / fiber_block / inf_norm (solver.py:162-192)."""
    from paper_2108_10448_b200 import DenseTensorAccessor

    shape = (7, 5, 6, 4)
    rng = np.random.default_rng(9)
    xf = rng.standard_normal(int(np.prod(shape)))
    acc = DenseTensorAccessor(DenseTensor(xf, shape))
    arr = xf.reshape(shape, order="F")
    rows = tuple(np.sort(rng.choice(d, s, replace=False)) + 1 for d, s in zip(shape, (3, 2, 4, 1)))
    np.testing.assert_array_equal(acc.core_block(rows), orc.core_block(arr, rows))
    for k in range(1, 5):
        tot = int(np.prod(shape)) // shape[k - 1]
        cols = np.sort(rng.choice(tot, 9, replace=False)) + 1
        np.testing.assert_array_equal(acc.fiber_block(k, cols), orc.gather_fibers(xf, shape, k, cols))
    assert acc.inf_norm() == float(np.max(np.abs(xf)))
    with pytest.raises(IndexError):
        acc.core_block((np.array([8]), np.array([1]), np.array([1]), np.array([1])))


def test_phase_timings_from_device_events():
    from paper_2108_10448_b200 import solver as solver_mod

    shape, ranks = (30, 24, 20), (2, 2, 2)
    rows, cols = baseline_sample_sizes(shape, ranks)
    xf, _, _ = make_gaussian_tucker(shape, ranks, 0.15, 10.0, seed=8)
    cfg = SolverConfig(ranks=ranks, eps=1e-5, variant="R", max_iters=40, seed=2, row_sample_sizes=rows,
                       col_sample_sizes=cols)
    base = rtcur(DenseTensor(xf, shape), cfg)
    assert base.timings["timing_source"] == "host"
    solver_mod.PHASE_TIMINGS = True
    try:
        res = rtcur(DenseTensor(xf, shape), cfg)
    finally:
        solver_mod.PHASE_TIMINGS = False
    t = res.timings
    assert t["timing_source"] == "device-events"
    assert set(t) >= {"sample", "gather", "eval_lowrank", "threshold", "build", "error", "total"}
    for key in ("gather", "eval_lowrank", "threshold", "build", "error"):
        assert t[key] > 0.0, key
    assert res.error_history == base.error_history


@pytest.mark.parametrize("shape,r", [((213, 3017), 10), ((174, 1999), 10), ((165, 900), 7), ((220, 2100), 4),
                                     ((140, 5000), 12), ((90, 2693), 5)])
def test_truncated_svd_cluster_sizes_vs_oracle(shape, r):
    """Intersections with 128 < s <= 256 take the cluster (8 CTAs, registers)
    tridiagonalisation: the rank-r truncated SVD through the kernel plug matches
    the oracle's Golub-Kahan-Reinsch SVD (reconstruction 1e-10 x sigma_1)."""
    rng = np.random.default_rng(sum(shape) + r)
    m, p = shape
    # decaying spectrum + noise floor, like a cleaned intersection
    q1, _ = np.linalg.qr(rng.standard_normal((m, m)))
    q2, _ = np.linalg.qr(rng.standard_normal((p, m)))
    sv = np.concatenate([np.geomspace(100.0, 10.0, r), np.geomspace(3.0, 0.01, m - r)])
    mat = (q1 * sv) @ q2.T
    want = orc.truncated_svd(mat, r)
    lib = _native.load()
    st = torch.cuda.current_stream().cuda_stream
    a = torch.from_numpy(np.asfortranarray(mat).reshape(-1, order="F").copy()).cuda()
    u = torch.empty(m * r, dtype=torch.float64, device="cuda")
    v = torch.empty(p * r, dtype=torch.float64, device="cuda")
    s = torch.empty(r, dtype=torch.float64, device="cuda")
    _native.check(lib.rtcur_truncated_svd(a.data_ptr(), m, p, r, u.data_ptr(), s.data_ptr(), v.data_ptr(), st))
    U = u.cpu().numpy().reshape((m, r), order="F")
    V = v.cpu().numpy().reshape((p, r), order="F")
    S = s.cpu().numpy()
    np.testing.assert_allclose(S, want.singular_values, rtol=0, atol=1e-12 * sv[0])
    np.testing.assert_allclose((U * S) @ V.T, want.reconstruct(), rtol=0, atol=1e-10 * sv[0])
    np.testing.assert_allclose(U.T @ U, np.eye(r), atol=1e-12)
