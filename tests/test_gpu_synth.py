"""The reference generator's semantics on the device against
instances made by the real reference (tests/golden/synth_instances.npz)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return load_golden("synth_instances.npz")


def test_make_instance_device_matches_reference(golden):
    from paper_2108_10448_b200.synth import InstanceSpec, make_instance_device

    for i, (n, d, r, a, s) in enumerate(golden["specs"]):
        spec = InstanceSpec(int(n), int(d), int(r), float(a), int(s))
        x, low, sparse = make_instance_device(spec)
        assert x.shape == spec.shape
        lo, sp, xx = low.flat.cpu().numpy(), sparse.flat.cpu().numpy(), x.flat.cpu().numpy()
        ref_low, ref_sp, ref_x = golden[f"low{i}"], golden[f"sparse{i}"], golden[f"x{i}"]
        scale = np.max(np.abs(ref_low))
        # low-rank part: same draws, expansion order differs -> a few ulps of max|L|
        np.testing.assert_allclose(lo, ref_low, rtol=0, atol=1e-13 * scale)
        # outlier support: bit-exact positions (same sampler stream)
        assert np.array_equal(sp != 0, ref_sp != 0), i
        assert int(np.count_nonzero(sp)) == int(np.floor(a * spec.shape[0] ** spec.n + 1e-9))
        # values: same uniforms, mu = mean|L| to ~1 ulp
        np.testing.assert_allclose(sp, ref_sp, rtol=1e-12, atol=0)
        np.testing.assert_allclose(xx, ref_x, rtol=0, atol=1e-12 * max(scale, np.max(np.abs(ref_sp), initial=0)))
        assert np.array_equal(xx[sp == 0], lo[sp == 0])


def test_generator_validation():
    from paper_2108_10448_b200.synth import InstanceSpec

    with pytest.raises(ValueError):
        InstanceSpec(3, 5, 9, 0.1, 0)
    with pytest.raises(ValueError):
        InstanceSpec(3, 5, 2, 1.0, 0)
