"""Streamed TNSR I/O between disk and HBM, and the `rtcur solve` output set
(cli.py:148-273 mirror) against the reference's golden solves."""

import json
import os

import numpy as np
import pytest

from conftest import golden_cfg_kwargs, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


def _host(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(int(np.prod(shape)))


def test_device_read_f64_f32_and_slab(torch, tmp_path):
    from paper_2108_10448_b200.tensor import DenseTensor
    from paper_2108_10448_b200.tensorfile import read_tensor_device, write_tensor

    shape = (37, 11, 5)
    flat = _host(shape, 1)
    p = tmp_path / "x.tnsr"
    write_tensor(p, DenseTensor(flat, shape))
    x = read_tensor_device(p)
    assert x.shape == shape and x.flat.dtype == torch.float64
    assert np.array_equal(x.flat.cpu().numpy(), flat)
    x32 = read_tensor_device(p, dtype=torch.float32)
    assert np.array_equal(x32.flat.cpu().numpy(), flat.astype(np.float32))
    arr = flat.reshape(shape, order="F")
    for lo, hi in ((0, 9), (9, 18), (30, 37)):
        s = read_tensor_device(p, slab=(lo, hi))
        assert s.shape == (hi - lo, 11, 5)
        assert np.array_equal(s.flat.cpu().numpy(), arr[lo:hi].reshape(-1, order="F"))


def test_device_write_matches_host_writer(torch, tmp_path):
    from paper_2108_10448_b200.tensor import DenseTensor, DeviceTensor
    from paper_2108_10448_b200.tensorfile import write_tensor, write_tensor_device

    shape = (6, 7, 8)
    flat = _host(shape, 2)
    a, b = tmp_path / "a.tnsr", tmp_path / "b.tnsr"
    write_tensor(a, DenseTensor(flat, shape))
    write_tensor_device(b, DeviceTensor(torch.from_numpy(flat).cuda(), shape))
    assert a.read_bytes() == b.read_bytes()
    c = tmp_path / "c.tnsr"   # fp32 device data widens exactly
    f32 = flat.astype(np.float32)
    write_tensor_device(c, DeviceTensor(torch.from_numpy(f32).cuda(), shape))
    d = tmp_path / "d.tnsr"
    write_tensor(d, DenseTensor(f32.astype(np.float64), shape))
    assert c.read_bytes() == d.read_bytes()


def test_multi_chunk_round_trip(torch, tmp_path):
    # 200 MB payload: several 64 MB staging chunks in both directions
    from paper_2108_10448_b200.tensor import DeviceTensor
    from paper_2108_10448_b200.tensorfile import read_header, read_tensor_device, write_tensor_device

    shape = (125, 400, 500)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = DeviceTensor(torch.randn(int(np.prod(shape)), dtype=torch.float64, device="cuda", generator=g), shape)
    p = tmp_path / "big.tnsr"
    write_tensor_device(p, x)
    assert read_header(p) == (1, shape)
    assert os.path.getsize(p) == 8 + 8 * 3 + 8 * int(np.prod(shape))
    y = read_tensor_device(p)
    assert torch.equal(x.flat, y.flat)
    s = read_tensor_device(p, dtype=torch.float32, slab=(40, 85))
    ref = x.flat.reshape(500, 400, 125)[:, :, 40:85].contiguous().reshape(-1).float()
    assert torch.equal(s.flat, ref)


@pytest.mark.parametrize("case", ["d20_F", "bern_R", "n4_R"])
def test_solve_to_dir_matches_reference(torch, tmp_path, case):
    from paper_2108_10448_b200.cli import solve_to_dir
    from paper_2108_10448_b200.tensor import DenseTensor
    from paper_2108_10448_b200.tensorfile import read_tensor, write_tensor

    g = load_golden(f"solve_{case}.npz")
    shape = tuple(int(v) for v in g["shape"])
    p = tmp_path / "X.tnsr"
    write_tensor(p, DenseTensor(g["x"], shape))
    kw = golden_cfg_kwargs(g)
    if "row_sample_sizes" in kw:
        pytest.skip("explicit sample sizes are not a solve CLI option")
    out = tmp_path / "run"
    code = solve_to_dir(str(p), str(out), kw["ranks"], upsilon=kw["upsilon"], gamma=kw["gamma"], zeta0=kw["zeta0"],
                        eps=kw["eps"], variant=kw["variant"], max_iters=kw["max_iters"], seed=kw["seed"] or 0,
                        full_output=True)
    assert code == (0 if bool(g["converged"]) else 3)
    hist = (out / "error_history.csv").read_text().strip().split("\n")
    assert hist[0] == "iteration,e"
    got = np.array([float(line.split(",")[1]) for line in hist[1:]])
    np.testing.assert_allclose(got, g["error_history"], rtol=0, atol=1e-10)
    idx = json.loads((out / "indices.json").read_text())
    for m in range(len(shape)):
        assert idx["rows"][m] == g[f"rows{m}"].tolist() and idx["cols"][m] == g[f"cols{m}"].tolist()
    L = read_tensor(out / "L.tnsr")
    S = read_tensor(out / "S.tnsr")
    np.testing.assert_allclose(L.data, g["full_L"].reshape(-1, order="F"), rtol=0, atol=1e-10)
    assert np.array_equal(S.data != 0, g["full_S"].reshape(-1, order="F") != 0)
    np.testing.assert_allclose(S.data, g["full_S"].reshape(-1, order="F"), rtol=0, atol=1e-10)
    for m in range(len(shape)):
        fac = read_tensor(out / f"factor_mode{m + 1}.tnsr").data.reshape(g[f"cur_factor{m}"].shape, order="F")
        np.testing.assert_allclose(fac, g[f"cur_factor{m}"], rtol=0, atol=1e-8)
    man = dict(line.split(": ", 1) for line in (out / "manifest.txt").read_text().strip().split("\n"))
    assert man["command"] == "solve" and man["iterations"] == str(int(g["iterations"]))
    assert man["outputs"].split(",")[-2:] == ["L.tnsr", "S.tnsr"]


def test_full_output_cap_and_missing_input(torch, tmp_path, monkeypatch):
    from paper_2108_10448_b200 import cli

    assert cli.solve_to_dir(str(tmp_path / "absent.tnsr"), str(tmp_path / "o"), (1, 1)) == cli.DATA_ERROR
    from paper_2108_10448_b200.tensor import DenseTensor
    from paper_2108_10448_b200.tensorfile import write_tensor

    p = tmp_path / "x.tnsr"
    write_tensor(p, DenseTensor(np.ones(60), (3, 4, 5)))
    monkeypatch.setattr(cli, "FULL_OUTPUT_CAP", 10)
    with pytest.raises(cli.UsageError, match="cap 10"):
        cli.solve_to_dir(str(p), str(tmp_path / "o"), (1, 1, 1), full_output=True)
    with pytest.raises(cli.UsageError, match="2 entries for a 3-mode"):
        cli.solve_to_dir(str(p), str(tmp_path / "o"), (1, 1))
