"""CPU-only tests: host logic of the drop-in (sampling, config, helpers) and
the C-ABI library surface (loads, exports every symbol of include/*.h).
No compute call needs a GPU here."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2108_10448_b200 import SolverConfig, sample_sizes, sampled_relative_error, zeta_schedule
from paper_2108_10448_b200 import fiber_cur as fc
from paper_2108_10448_b200 import _native
from paper_2108_10448_b200.synth import CONFIGS, baseline_sample_sizes
from paper_2108_10448_b200.tensor import DenseTensor, decode_fiber_columns, fiber_base_offsets, mode_stride


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "rtcur_b200.h")).read()
    return sorted(set(re.findall(r"\b(rtcur_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTED)
    _native.load()
    assert b"sm_100a" in _native.load().rtcur_version()


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_mapping():
    _native.load()
    with pytest.raises(ValueError):
        _native.check(_native.RTCUR_E_VALUE)
    with pytest.raises(IndexError):
        _native.check(_native.RTCUR_E_INDEX)
    with pytest.raises(ArithmeticError):
        _native.check(_native.RTCUR_E_ARITH)
    with pytest.raises(RuntimeError):
        _native.check(_native.RTCUR_E_CUDA)


def test_engine_plan_sizes_and_errors():
    lib = _native.load()
    ws, xo, xn = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    for cfg in CONFIGS.values():
        rows, cols = baseline_sample_sizes(cfg.shape, cfg.ranks)
        n = len(cfg.shape)
        st = lib.rtcur_engine_plan(n, _native.i64_array(cfg.shape), _native.i32_array(cfg.ranks),
                                   _native.i64_array(rows), _native.i64_array(cols), 1, ctypes.byref(ws),
                                   ctypes.byref(xo), ctypes.byref(xn))
        assert st == 0, _native.load().rtcur_last_error()
        nblk = int(np.prod(rows)) + sum(d * c for d, c in zip(cfg.shape, cols))
        assert nblk <= xn.value <= nblk + 3 * len(cfg.shape)   # fiber blocks start 16-byte aligned
        assert ws.value < 8 * 2 ** 30
    # rank above the sample sizes -> ValueError (fiber_cur.py:257-261)
    st = lib.rtcur_engine_plan(3, _native.i64_array((10, 10, 10)), _native.i32_array((3, 3, 3)),
                               _native.i64_array((2, 5, 5)), _native.i64_array((5, 5, 5)), 0, ctypes.byref(ws),
                               ctypes.byref(xo), ctypes.byref(xn))
    with pytest.raises(ValueError):
        _native.check(st)


def test_sampler_matches_reference_golden(kernels_golden):
    g = kernels_golden
    i = 0
    while f"draw{i}_shape" in g:
        shape = tuple(int(d) for d in g[f"draw{i}_shape"])
        rng = np.random.default_rng(int(g[f"draw{i}_seed"]))
        idx = fc.draw_sample_indices(shape, g[f"draw{i}_rs"], g[f"draw{i}_cs"], rng)
        for m in range(len(shape)):
            assert np.array_equal(idx.rows[m], g[f"draw{i}_rows{m}"])
            assert np.array_equal(idx.cols[m], g[f"draw{i}_cols{m}"])
        idx2 = fc.draw_sample_indices(shape, g[f"draw{i}_rs"], g[f"draw{i}_cs"], rng)
        for m in range(len(shape)):
            assert np.array_equal(idx2.cols[m], g[f"draw{i}_cols{m}_second"])
        i += 1


def test_sample_sizes_golden(kernels_golden):
    g = kernels_golden
    i = 0
    while f"sizes{i}_shape" in g:
        rows, cols = sample_sizes(tuple(g[f"sizes{i}_shape"]), tuple(g[f"sizes{i}_ranks"]), float(g[f"sizes{i}_ups"]))
        assert rows == tuple(g[f"sizes{i}_rows"]) and cols == tuple(g[f"sizes{i}_cols"])
        i += 1
    with pytest.raises(ValueError):
        sample_sizes((10, 10), (3, 3), 0.0)
    with pytest.raises(ValueError):
        sample_sizes((10, 10), (11, 3), 2.0)


def test_baseline_sizes_match_survey_table():
    # |I| = ceil(3 r ln d) (clamped), |J| = ceil(3 r^2 ln^2 d)
    want = {0: ((42,) * 3, (573,) * 3), 1: ((90,) * 3, (2693,) * 3), 2: ((213,) * 3, (15081,) * 3),
            3: ((165, 174, 3, 39), (9012, 9983, 33, 492)), 4: ((65,) * 4, (1397,) * 4)}
    for i, (rows, cols) in want.items():
        c = CONFIGS[i]
        assert baseline_sample_sizes(c.shape, c.ranks) == (rows, cols)


def test_config_validation_mirrors_reference():
    good = SolverConfig(ranks=(2, 2), gamma=0.5)
    assert good.variant == "F"
    for bad in (dict(gamma=1.0), dict(gamma=0.0), dict(eps=0.0), dict(zeta0=-1.0), dict(variant="x"),
                dict(max_iters=0), dict(upsilon=0.0)):
        with pytest.raises(ValueError):
            SolverConfig(ranks=(2, 2), **bad)
    with pytest.raises(ValueError):
        SolverConfig(ranks=(0, 2))
    assert SolverConfig(ranks=(2, 2), variant="r").variant == "R"
    cfg = SolverConfig(ranks=(2, 2, 2), upsilon=3.0, row_sample_sizes=(5, 5, 5))
    rows, cols = cfg.resolve_sample_sizes((30, 30, 30))
    assert rows == (5, 5, 5)
    assert cols == tuple(min(900, max(2, int(np.ceil(6 * np.log(900))))) for _ in range(3))


def test_zeta_and_error_helpers():
    assert zeta_schedule(255.0, 0.7, 1) == pytest.approx(178.5, abs=1e-12)
    assert zeta_schedule(1.0, 0.7, 10) == pytest.approx(0.0282475249, abs=1e-10)
    with pytest.raises(ValueError):
        zeta_schedule(1.0, 0.7, -1)
    z = np.zeros((2, 2))
    assert sampled_relative_error(z, [z], np.ones((2, 2)), [np.ones((2, 2))]) == 0.0
    assert sampled_relative_error(z, [z], z, [z]) == 0.0
    assert sampled_relative_error(np.ones((2, 2)), [z], z, [z]) == float("inf")
    from paper_2108_10448_b200.solver import _error_from_sums

    assert _error_from_sums([0.0, 0.0], [0.0, 0.0]) == 0.0
    assert _error_from_sums([1.0, 0.0], [0.0, 0.0]) == float("inf")
    assert _error_from_sums([4.0, 9.0], [16.0, 9.0]) == pytest.approx(5.0 / 7.0)


def test_layout_helpers():
    assert mode_stride((3, 4, 5), 3) == 12
    parts = decode_fiber_columns((3, 4, 5), 2, np.array([1, 3, 15]))
    assert [list(p) for p in parts] == [[1, 3, 3], [1, 1, 5]]
    assert list(fiber_base_offsets((3, 4, 5), 2, np.array([1, 3, 15]))) == [0, 2, 50]
    with pytest.raises(IndexError):
        decode_fiber_columns((3, 4, 5), 2, np.array([16]))
    t = DenseTensor(np.arange(24.0), (2, 3, 4))
    assert t.value_at((2, 3, 4)) == 23.0
    assert t.data.flags.writeable is False


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2108_10448_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "rtcur_oracle" not in src and "liboracle" not in src, f
