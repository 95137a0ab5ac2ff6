"""TNSR v1 host API vs the reference's golden bytes and error texts
(tests/golden/tnsr_golden.json, made by make_tnsr_golden.py from the real
reference; cases mirror /root/reference/pkg/tests/test_tensorfile.py)."""

import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2108_10448_b200.tensor import DenseTensor
from paper_2108_10448_b200.tensorfile import (FORMAT_VERSION, MAGIC, TensorFormatError, read_header, read_tensor,
                                              write_tensor)


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "tnsr_golden.json")) as f:
        return json.load(f)


def test_constants():
    assert MAGIC == b"TNSR" and FORMAT_VERSION == 1


def test_writer_bytes_match_reference(golden, tmp_path):
    for i, case in enumerate(golden["written"]):
        raw = bytes.fromhex(case["hex"])
        shape = tuple(case["shape"])
        n = len(shape)
        vals = np.frombuffer(raw[8 + 8 * n:], dtype="<f8")
        p = tmp_path / f"w{i}.tnsr"
        write_tensor(p, DenseTensor._wrap(np.reshape(vals.copy(), shape, order="F")))
        assert p.read_bytes() == raw


def test_reader_on_reference_files(golden, tmp_path):
    for i, case in enumerate(golden["headers"]):
        raw = bytes.fromhex(case["hex"])
        p = tmp_path / f"h{i}.tnsr"
        p.write_bytes(raw)
        v, dims = read_header(p)
        assert v == case["version"] and list(dims) == case["dims"]
        t = read_tensor(p)
        n = len(dims)
        assert t.shape == tuple(dims)
        assert np.array_equal(t.data, np.frombuffer(raw[8 + 8 * n:], dtype="<f8"), equal_nan=True)


def test_error_texts_match_reference(golden, tmp_path):
    for case in golden["errors"]:
        p = tmp_path / f"{case['name']}.tnsr"
        p.write_bytes(bytes.fromhex(case["hex"]))
        with pytest.raises(TensorFormatError) as exc:
            read_tensor(p)
        assert str(exc.value) == case["message"].replace("{path}", str(p)), case["name"]
        assert isinstance(exc.value, ValueError)


def test_special_values_survive(tmp_path):
    t = DenseTensor([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-308], (6,))
    p = tmp_path / "t.tnsr"
    write_tensor(p, t)
    back = read_tensor(p)
    assert np.array_equal(back.data, t.data, equal_nan=True)
    assert np.signbit(back.data[1])


def test_payload_is_layout_order(tmp_path):
    t = DenseTensor([1, 2, 3, 4, 5, 6], (2, 3))
    p = tmp_path / "t.tnsr"
    write_tensor(p, t)
    raw = p.read_bytes()
    header = MAGIC + struct.pack("<HH", 1, 2) + struct.pack("<QQ", 2, 3)
    assert raw[:len(header)] == header
    assert np.array_equal(np.frombuffer(raw[len(header):], dtype="<f8"), [1, 2, 3, 4, 5, 6])


def test_missing_file(tmp_path):
    with pytest.raises(FileNotFoundError):
        read_tensor(tmp_path / "absent.tnsr")
    with pytest.raises(FileNotFoundError):
        read_header(tmp_path / "absent.tnsr")


def test_round_trip_property(tmp_path):
    rng = np.random.default_rng(7)
    for i in range(100):
        n = int(rng.integers(1, 5))
        shape = tuple(int(rng.integers(1, 6)) for _ in range(n))
        t = DenseTensor(rng.standard_normal(int(np.prod(shape))), shape)
        p = tmp_path / f"p{i}.tnsr"
        write_tensor(p, t)
        back = read_tensor(p)
        assert back.shape == shape
        assert np.array_equal(back.data, t.data)


@pytest.mark.parametrize("dims", [(2 ** 32,) * 4, (2 ** 63 - 1, 3), (2 ** 64 - 1,), (2 ** 40, 2 ** 40, 2 ** 40)])
def test_huge_extents_rejected_like_reference(tmp_path, dims):
    """A header whose extents overflow 64/128-bit products must fail the payload
    check with the reference's exact text (Python-int product,
    tensorfile.py:94-108), never wrap to a small size."""
    p = tmp_path / "huge.tnsr"
    p.write_bytes(MAGIC + struct.pack("<HH", FORMAT_VERSION, len(dims)) + struct.pack(f"<{len(dims)}Q", *dims))
    count = 1
    for d in dims:
        count *= d
    with pytest.raises(TensorFormatError) as exc:
        read_tensor(p)
    assert str(exc.value) == (f"{p}: payload at byte {8 + 8 * len(dims)} holds 0 bytes, dims {tuple(dims)} "
                              f"require {count * 8}")
