"""Dense HOSVD-AP baseline on the GPU vs the real reference's
ap_hosvd_trpca on the same instances (tests/golden/ap_hosvd.npz)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return load_golden("ap_hosvd.npz")


def test_ap_hosvd_matches_reference(golden):
    import torch

    from paper_2108_10448_b200.hosvd_ap import ap_hosvd_trpca
    from paper_2108_10448_b200.tensor import DeviceTensor

    for i, (n, d, r, a, s, tz, mi) in enumerate(golden["cases"]):
        n, d, r, mi = int(n), int(d), int(r), int(mi)
        shape = (d,) * n
        x = DeviceTensor(torch.from_numpy(golden[f"x{i}"]).cuda(), shape)
        z = float(golden[f"zeta0_{i}"])
        L, S, hist = ap_hosvd_trpca(x, (r,) * n, zeta0=None if np.isnan(z) else z, gamma=0.7, eps=1e-5, max_iters=mi)
        ref = golden[f"hist{i}"]
        assert len(hist) == len(ref), (i, len(hist), len(ref))
        np.testing.assert_allclose(hist, ref, rtol=1e-8, atol=1e-12)
        np.testing.assert_allclose(L.flat.cpu().numpy(), golden[f"L{i}"], rtol=0, atol=1e-9)
        Sg = S.flat.cpu().numpy()
        assert np.array_equal(Sg != 0, golden[f"S{i}"] != 0)
        np.testing.assert_allclose(Sg, golden[f"S{i}"], rtol=0, atol=1e-9)


def test_ap_hosvd_validation(golden):
    from paper_2108_10448_b200.hosvd_ap import ap_hosvd_trpca
    from paper_2108_10448_b200.tensor import DenseTensor

    x = DenseTensor(np.ones(8), (2, 2, 2))
    with pytest.raises(ValueError):
        ap_hosvd_trpca(x, (1, 1), gamma=0.7)
    with pytest.raises(ValueError):
        ap_hosvd_trpca(x, (1, 1, 1), gamma=1.5)
    with pytest.raises(ValueError):
        ap_hosvd_trpca(x, (3, 1, 1))
