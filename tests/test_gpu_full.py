"""GPU: the full-output step K3 (cli.py:237-243 -- L = cur_reconstruct_full,
S = hard_threshold(x - L, zeta_final)) on its two device paths.

k_full_tma (TMA-staged, A_1 rows in registers) must be bit-identical per
element to the generic grid-stride k_full (same FMA order), which the golden
solves in test_gpu_parity.py pin against the reference; both are checked here
against a numpy Tucker reconstruction of the exported FiberCur
(fiber_cur.py:277-285).  The shapes walk the TMA planner's envelope: 16- and
8-byte vectors (fp32 ranks <= 8 / > 8, fp64), one and several row bands,
several fibers per thread row (short mode 1), ranks up to 16, the
X-less reconstruction, and an odd mode-1 length that falls back to k_full.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, run on the B200
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_10448_b200 import DeviceTensor, SolverConfig, full_output, rtcur  # noqa: E402
from paper_2108_10448_b200.full import cur_reconstruct_full  # noqa: E402
from paper_2108_10448_b200.synth import baseline_sample_sizes, make_gaussian_tucker  # noqa: E402

CASES = [
    # shape, ranks, dtype
    ((40, 36, 30), (3, 3, 3), np.float32),     # 16-byte vectors, one band
    ((44, 20, 18), (5, 4, 4), np.float64),     # fp64 double2
    ((2000, 6, 5), (2, 2, 2), np.float32),     # two row bands (> 384 x 4 rows)
    ((800, 12, 10), (3, 3, 3), np.float64),    # two row bands (> 384 x 2 rows)
    ((28, 30, 26), (4, 4, 4), np.float32),     # short fibers: several per thread row
    ((64, 40, 30), (10, 4, 4), np.float32),    # rank > 8: 8-byte vectors
    ((48, 30, 30), (16, 3, 3), np.float64),    # rank 16
    ((27, 30, 26), (3, 3, 3), np.float32),     # odd mode-1 length -> generic k_full
    ((30, 20, 12, 10), (3, 2, 2, 2), np.float32),   # 4 modes
]


def _solve(shape, ranks, dtype):
    xf, _, _ = make_gaussian_tucker(shape, ranks, 0.2, 10.0, seed=7, dtype=dtype)
    rows, cols = baseline_sample_sizes(shape, ranks)
    cfg = SolverConfig(ranks=ranks, eps=1e-5, variant="F", max_iters=4, seed=2, row_sample_sizes=rows,
                       col_sample_sizes=cols)
    dev = DeviceTensor(torch.from_numpy(xf).cuda(), shape)
    return xf, dev, rtcur(dev, cfg)


def _generic(fn):
    os.environ["RTCUR_K3_GENERIC"] = "1"
    try:
        return fn()
    finally:
        del os.environ["RTCUR_K3_GENERIC"]


def _tucker(cur, shape):
    """fiber_cur.py:277-285 in numpy: core x_i factors[i]."""
    t = np.asarray(cur.core.data).reshape([len(r) for r in cur.indices.rows], order="F")
    for m, f in enumerate(cur.factors):
        t = np.moveaxis(np.tensordot(f, t, axes=([1], [m])), 0, m)
    return t.reshape(-1, order="F")


@pytest.mark.parametrize("shape,ranks,dtype", CASES, ids=[f"{'x'.join(map(str, c[0]))}-r{c[1][0]}-{np.dtype(c[2]).name}"
                                                         for c in CASES])
def test_k3_tma_matches_generic_and_tucker(shape, ranks, dtype):
    xf, dev, res = _solve(shape, ranks, dtype)
    L1, S1, rel1 = full_output(res, dev)
    L2, S2, rel2 = _generic(lambda: full_output(res, dev))
    assert torch.equal(L1.flat, L2.flat)
    assert torch.equal(S1.flat, S2.flat)
    assert rel1 == pytest.approx(rel2, rel=1e-12, abs=1e-300)
    want = _tucker(res.cur, shape)
    got = L1.flat.double().cpu().numpy()
    tol = 1e-10 if dtype == np.float64 else 1e-6
    assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want)
    # S = HT(x - L, zeta_final), strict keep (py_kernels.py:226-230)
    x = xf.astype(np.float64)
    s_got = S1.flat.double().cpu().numpy()
    d = x - got
    s_want = np.where(np.abs(d) > res.zeta_final, d, 0.0)
    if dtype == np.float64:   # L is stored exactly: S follows bit-exactly
        assert np.array_equal(s_got, s_want)
    else:                     # L was rounded to fp32 on store: exact away from the threshold
        far = np.abs(np.abs(d) - res.zeta_final) > 1e-5 * max(res.zeta_final, 1e-30) + 1e-6 * np.abs(x)
        assert np.array_equal((s_got != 0)[far], (s_want != 0)[far])
        np.testing.assert_allclose(s_got[far], s_want[far], rtol=1e-6, atol=1e-6 * float(np.abs(x).max()))
    # X-less reconstruction (cur_reconstruct_full) takes the same path
    Lh = cur_reconstruct_full(res.cur).data
    Lg = _generic(lambda: cur_reconstruct_full(res.cur).data)
    assert np.array_equal(np.asarray(Lh), np.asarray(Lg))

