"""Pin the CPU oracle against vectors recorded from the real reference.

The fixtures in tests/golden were produced by tests/golden/make_golden.py,
which imports /root/reference (scratch build, compiled backend).  Bars are
the reference's own: indices and hard threshold bit-exact,
S/L blocks and errors 1e-10 (test_reference.py:177-214), singular values
1e-12*scale and reconstructions 1e-10*scale (test_backends.py:46-71).
"""

import numpy as np
import pytest

from conftest import golden_cfg_kwargs, load_golden, solve_cases
from oracle import rtcur_oracle as orc


def test_sample_sizes_known_answers(kernels_golden):
    g = kernels_golden
    i = 0
    while f"sizes{i}_shape" in g:
        rows, cols = orc.sample_sizes(tuple(g[f"sizes{i}_shape"]), tuple(g[f"sizes{i}_ranks"]),
                                      float(g[f"sizes{i}_ups"]))
        assert rows == tuple(g[f"sizes{i}_rows"])
        assert cols == tuple(g[f"sizes{i}_cols"])
        i += 1
    assert i >= 5
    # reference worked examples (test_fiber_cur.py:39-59)
    assert orc.sample_sizes((300, 300, 300), (3, 3, 3), 3.0) == ((52,) * 3, (103,) * 3)


def test_draws_bit_exact(kernels_golden):
    g = kernels_golden
    i = 0
    while f"draw{i}_shape" in g:
        shape = tuple(int(d) for d in g[f"draw{i}_shape"])
        rng = np.random.default_rng(int(g[f"draw{i}_seed"]))
        idx = orc.draw_sample_indices(shape, g[f"draw{i}_rs"], g[f"draw{i}_cs"], rng)
        for m in range(len(shape)):
            assert np.array_equal(idx.rows[m], g[f"draw{i}_rows{m}"])
            assert np.array_equal(idx.cols[m], g[f"draw{i}_cols{m}"])
        idx2 = orc.draw_sample_indices(shape, g[f"draw{i}_rs"], g[f"draw{i}_cs"], rng)
        for m in range(len(shape)):
            assert np.array_equal(idx2.cols[m], g[f"draw{i}_cols{m}_second"])
        i += 1
    assert i >= 6


def test_hard_threshold_bit_exact(kernels_golden):
    g = kernels_golden
    for i in range(6):
        y = orc.hard_threshold(g[f"ht{i}_x"], float(g[f"ht{i}_z"]))
        assert np.array_equal(y, g[f"ht{i}_y"])
    assert np.array_equal(orc.hard_threshold(g["ht_edge_x"], 1.0), g["ht_edge_y"])
    with pytest.raises(ValueError):
        orc.hard_threshold(np.ones(3), -0.1)


def test_gather_bit_exact(kernels_golden):
    g = kernels_golden
    for i in range(5):
        flat = g[f"gather{i}_flat"]
        bases = g[f"gather{i}_bases"]
        stride, length = int(g[f"gather{i}_stride"]), int(g[f"gather{i}_length"])
        idx = bases[None, :] + stride * np.arange(length)[:, None]
        assert np.array_equal(flat[idx], g[f"gather{i}_out"])


def test_svd_battery(kernels_golden):
    g = kernels_golden
    i = 0
    while f"svd{i}_m" in g:
        m, r = g[f"svd{i}_m"], int(g[f"svd{i}_r"])
        f = orc.truncated_svd(m, r)
        scale = max(float(g[f"svd{i}_s"][0]), 1.0)
        np.testing.assert_allclose(f.singular_values, g[f"svd{i}_s"], atol=1e-12 * scale)
        np.testing.assert_allclose(f.reconstruct(), g[f"svd{i}_rec"], atol=1e-10 * scale)
        np.testing.assert_allclose(f.pinv(), g[f"svd{i}_pinv"], atol=1e-8 * max(scale, 1.0 / scale))
        np.testing.assert_allclose(f.u.T @ f.u, np.eye(r), atol=1e-10)
        np.testing.assert_allclose(f.v.T @ f.v, np.eye(r), atol=1e-10)
        i += 1
    assert i >= 10


def test_svd_matches_lapack_wide_and_tall():
    rng = np.random.default_rng(5)
    for shape in [(7, 40), (40, 7), (1, 5), (5, 1), (33, 33)]:
        a = rng.standard_normal(shape)
        u, s, vt = orc.dense_svd(a)
        np.testing.assert_allclose(s, np.linalg.svd(a, compute_uv=False), rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose((u * s) @ vt, a, atol=1e-12)


def test_svd_errors():
    with pytest.raises(ValueError):
        orc.truncated_svd(np.ones((3, 4)), 0)
    with pytest.raises(ValueError):
        orc.truncated_svd(np.ones((3, 4)), 4)
    with pytest.raises(ValueError):
        orc.truncated_svd(np.array([[1.0, np.nan]]), 1)


@pytest.mark.parametrize("case", solve_cases())
def test_oracle_solve_matches_reference(case):
    g = load_golden(f"solve_{case}.npz")
    shape = tuple(int(d) for d in g["shape"])
    n = len(shape)
    kw = golden_cfg_kwargs(g)
    res = orc.solve(g["x"], shape, kw.pop("ranks"), record_trace=True, **kw)
    assert res.iterations == int(g["iterations"])
    assert res.converged == bool(g["converged"])
    np.testing.assert_allclose(res.error_history, g["error_history"], atol=1e-10, rtol=0)
    assert np.array_equal(np.array(res.diagnostics, dtype=bool).reshape(g["diagnostics"].shape), g["diagnostics"])
    assert res.zeta_final == pytest.approx(float(g["zeta_final"]), rel=1e-15)
    for m in range(n):
        assert np.array_equal(res.indices.rows[m], g[f"rows{m}"])
        assert np.array_equal(res.indices.cols[m], g[f"cols{m}"])
        sv = res.cur.intersections[m].singular_values
        np.testing.assert_allclose(sv, g[f"cur_sv{m}"], atol=1e-10 * max(1.0, float(g[f"cur_sv{m}"][0])))
        np.testing.assert_allclose(res.cur.factors[m] @ np.eye(res.cur.factors[m].shape[1]),
                                   g[f"cur_factor{m}"], atol=1e-8)
        np.testing.assert_allclose(res.s_fibers[m], g[f"s_fib{m}"], atol=1e-10)
        assert np.array_equal(res.s_fibers[m] != 0, g[f"s_fib{m}"] != 0)
    np.testing.assert_allclose(res.s_core.reshape(-1, order="F"), g["s_core"], atol=1e-10)
    assert np.array_equal(res.s_core.reshape(-1, order="F") != 0, g["s_core"] != 0)
    for t in g["trace_iters"]:
        tr = res.trace[int(t)]
        np.testing.assert_allclose(tr["s_core"].reshape(-1, order="F"), g[f"t{t}_s_core"], atol=1e-10)
        np.testing.assert_allclose(tr["l_core"].reshape(-1, order="F"), g[f"t{t}_l_core"], atol=1e-10)
        for m in range(n):
            np.testing.assert_allclose(tr["s_fibers"][m], g[f"t{t}_s_fib{m}"], atol=1e-10)
            np.testing.assert_allclose(tr["l_fibers"][m], g[f"t{t}_l_fib{m}"], atol=1e-10)
            assert np.array_equal(tr["indices"].cols[m], g[f"t{t}_cols{m}"])
    low, sp, _, _ = orc.full_output(g["x"], shape, res.cur, res.zeta_final)
    np.testing.assert_allclose(low, g["full_L"], atol=1e-8)
    np.testing.assert_allclose(sp, g["full_S"], atol=1e-8)


def test_oracle_cfg0_matches_reference_summary():
    """BASELINE config 0 (100^3, RTCUR-F, fp64) on the synth X."""
    from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config

    g = load_golden("cfg0_summary.npz")
    xf, _, _, bc = make_config(0)
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    res = orc.solve(xf, bc.shape, bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100,
                    seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols)
    assert res.iterations == int(g["iterations"])
    np.testing.assert_allclose(res.error_history, g["error_history"], atol=1e-10, rtol=0)
    s_core = res.s_core.reshape(-1, order="F")
    assert np.array_equal(np.packbits(s_core != 0), g["s_core_bits"])
    np.testing.assert_allclose(s_core[g["s_core_pos"]], g["s_core_val"], atol=1e-10)
    for m in range(3):
        s = res.s_fibers[m].reshape(-1, order="F")
        assert np.array_equal(np.packbits(s != 0), g[f"s_fib{m}_bits"])
        np.testing.assert_allclose(s[g[f"s_fib{m}_pos"]], g[f"s_fib{m}_val"], atol=1e-10)
        np.testing.assert_allclose(res.cur.intersections[m].singular_values, g[f"sv{m}"], rtol=1e-10)


def test_eval_fibers_blas_matches_einsum():
    """The BLAS-associated fiber evaluation the parity runs use equals the
    reference-shaped einsum (fiber_cur.py:318-326) to rounding, for 1-4 modes
    and column chunking."""
    rng = np.random.default_rng(11)
    for shape, isz in [((9,), (4,)), ((12, 7), (5, 3)), ((30, 20, 10), (6, 5, 4)),
                       ((11, 9, 7, 5), (4, 3, 5, 2))]:
        n = len(shape)
        core = np.asfortranarray(rng.standard_normal(isz))
        facs = tuple(rng.standard_normal((d, i)) for d, i in zip(shape, isz))
        cur = orc.OracleCur(core=core, fibers=tuple(np.zeros((d, 1)) for d in shape), intersections=(),
                            indices=None, factors=facs)
        for k in range(1, n + 1):
            tot = int(np.prod(shape)) // shape[k - 1]
            cols = np.sort(rng.choice(tot, min(tot, 23), replace=False)) + 1
            a = orc.eval_fibers_einsum(cur, k, cols)
            for chunk in (1 << 28, 64):
                b = orc.eval_fibers_blas(cur, k, cols, chunk_bytes=chunk)
                np.testing.assert_allclose(b, a, rtol=0, atol=1e-13 * max(1.0, np.abs(a).max()))


def test_oracle_einsum_and_blas_solves_agree():
    g = load_golden("solve_d10_R.npz")
    shape = tuple(int(d) for d in g["shape"])
    kw = golden_cfg_kwargs(g)
    ranks = kw.pop("ranks")
    a = orc.solve(g["x"], shape, ranks, eval_mode="einsum", **kw)
    b = orc.solve(g["x"], shape, ranks, eval_mode="blas", **kw)
    assert a.iterations == b.iterations
    np.testing.assert_allclose(a.error_history, b.error_history, atol=1e-13, rtol=0)
    np.testing.assert_array_equal(a.s_core != 0, b.s_core != 0)


def test_iter_solve_yields_reference_loop_state():
    """iter_solve's per-iteration state: zeta = gamma^k zeta0, S = HT(X - L_prev),
    error recomputed from the yielded blocks (solver.py:324-355)."""
    g = load_golden("solve_d10_F.npz")
    shape = tuple(int(d) for d in g["shape"])
    kw = golden_cfg_kwargs(g)
    ranks = kw.pop("ranks")
    zeta0 = orc.inf_norm(np.asarray(g["x"], dtype=np.float64)) if kw["zeta0"] is None else kw["zeta0"]
    for it in orc.iter_solve(g["x"], shape, ranks, **kw):
        k = it["iteration"]
        assert it["zeta"] == pytest.approx(kw["gamma"] ** k * zeta0, rel=1e-14)
        np.testing.assert_array_equal(it["s_core"], orc.hard_threshold(it["x_core"] - it["l_prev"][0], it["zeta"]))
        e_core = it["x_core"] - it["l_core"] - it["s_core"]
        e_f = [x - lf - s for x, lf, s in zip(it["x_fibers"], it["l_fibers"], it["s_fibers"])]
        assert orc.sampled_relative_error(e_core, e_f, it["x_core"], it["x_fibers"]) == it["error"]
        assert len(it["cur"].spectra) == len(shape)
        for m, inter in enumerate(it["cur"].intersections):
            np.testing.assert_array_equal(it["cur"].spectra[m][:ranks[m]], inter.singular_values)


def test_oracle_cfg1_matches_reference_summary():
    """BASELINE config 1 (400^3, RTCUR-R, fp64, the bench headline) solved by the
    oracle vs the REAL reference's run of the same instance
    (tests/golden/make_cfg1_golden.py): every iteration's index sets and S
    support per block (SHA-256), error (1e-10), S and L at fixed positions
    (1e-10); final singular values and the low-rank estimate at 2000 positions."""
    import hashlib

    from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config

    def sha(a):
        return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), dtype=np.uint8)

    g = load_golden("cfg1_summary.npz")
    xf, _, _, bc = make_config(1)
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    n = len(bc.shape)
    last = None
    k = 0
    for it in orc.iter_solve(xf, bc.shape, bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=100,
                             seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols):
        t = it["iteration"] - 1
        idx = it["indices"]
        assert np.array_equal(sha(np.concatenate([np.asarray(a, dtype=np.int64) for a in
                                                  list(idx.rows) + list(idx.cols)])), g[f"t{t}_idx_sha"])
        assert it["error"] == pytest.approx(float(g["error_history"][t]), abs=1e-10)
        assert it["zeta"] == pytest.approx(float(g[f"t{t}_zeta"]), rel=1e-15)
        sb = [it["s_core"].reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in it["s_fibers"]]
        lb = [it["l_core"].reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in it["l_fibers"]]
        for b in range(n + 1):
            assert np.array_equal(sha(np.packbits(sb[b] != 0.0)), g[f"t{t}_b{b}_supp_sha"]), (t, b)
            np.testing.assert_allclose(sb[b][g[f"pos{b}"]], g[f"t{t}_b{b}_s"], atol=1e-10, rtol=0)
            np.testing.assert_allclose(lb[b][g[f"pos{b}"]], g[f"t{t}_b{b}_l"], atol=1e-10, rtol=0)
        last = it
        k += 1
    assert k == int(g["iterations"])
    assert np.array_equal(np.packbits(last["s_core"].reshape(-1, order="F") != 0), g["s_core_bits"])
    for m in range(n):
        sv = last["cur"].intersections[m].singular_values
        np.testing.assert_allclose(sv, g[f"sv{m}"], rtol=1e-10)
    low = orc.reconstruct_full(last["cur"]).reshape(-1, order="F")
    np.testing.assert_allclose(low[g["L_pos"]], g["L_val"], atol=1e-10 * float(np.max(np.abs(g["L_val"]))))
