"""``rtcur solve`` outputs on the B200 path (mirror of the reference's
``cmd_solve``, /root/reference/pkg/src/rtcur/cli.py:148-273).

``solve_to_dir`` writes the same files with the same names, formats and
manifest keys as the reference command -- core/fibers/factors/sparse blocks as
TNSR files, indices.json, error_history.csv, manifest.txt and, with
``full_output``, L.tnsr / S.tnsr -- and returns the reference's exit code
(0 converged, 3 not converged, 2 unreadable input; ``UsageError`` for what the
reference reports as usage errors, including the full-output size cap of
cli.py:180-187).  The input is streamed from disk straight into HBM
(``read_tensor_device``) and the full L/S are written from HBM by the
streaming writer (``write_tensor_device``); argument parsing itself is out of
scope.
"""

from __future__ import annotations

import hashlib
import json
import os
import time

import numpy as np

from .solver import SolverConfig, rtcur
from .tensor import DenseTensor
from .tensorfile import TensorFormatError, read_header, read_tensor_device, write_tensor, write_tensor_device

__all__ = ["USAGE_ERROR", "DATA_ERROR", "NO_CONVERGENCE", "FULL_OUTPUT_CAP", "UsageError", "solve_to_dir"]

USAGE_ERROR = 1        # cli.py:39
DATA_ERROR = 2         # cli.py:40
NO_CONVERGENCE = 3     # cli.py:41
FULL_OUTPUT_CAP = 2 ** 31   # cli.py:45


class UsageError(ValueError):
    """What the reference reports on stderr with exit code 1 (cli.py _UsageError)."""


def _sha256(path) -> str:   # cli.py:58-63
    digest = hashlib.sha256()
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            digest.update(chunk)
    return digest.hexdigest()


def _fmt(value) -> str:     # cli.py:66-73
    if isinstance(value, bool):
        return "true" if value else "false"
    if isinstance(value, float):
        return repr(value)
    if isinstance(value, (tuple, list)):
        return ",".join(_fmt(v) for v in value)
    return str(value)


def _write_manifest(path, pairs) -> None:   # cli.py:76-79
    with open(path, "w") as f:
        for key, value in pairs:
            f.write(f"{key}: {_fmt(value)}\n")


def _write_matrix(path, mat) -> None:   # cli.py:143-144
    write_tensor(path, DenseTensor._wrap(np.asfortranarray(mat)))


def solve_to_dir(input_path, out_dir, ranks, *, upsilon=3.0, gamma=0.7, zeta0=None, eps=1e-5, variant="F",
                 max_iters=500, seed=0, full_output=False, force=False, dtype=None, stderr=None) -> int:
    """cmd_solve (cli.py:148-273) with the reference's defaults (cli.py:407-423)."""
    import sys

    import torch

    err = stderr or sys.stderr
    try:
        _, dims = read_header(input_path)
    except FileNotFoundError:
        print(f"error: cannot read {input_path}: no such file", file=err)
        return DATA_ERROR
    except (TensorFormatError, OSError) as exc:
        print(f"error: {exc}", file=err)
        return DATA_ERROR
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != len(dims):
        raise UsageError(f"--ranks has {len(ranks)} entries for a {len(dims)}-mode tensor")
    try:
        cfg = SolverConfig(ranks=ranks, eps=eps, zeta0=zeta0, gamma=gamma, upsilon=upsilon, variant=variant.upper(),
                           max_iters=max_iters, seed=seed)
        for m, (r, d) in enumerate(zip(cfg.ranks, dims), start=1):
            if r > d:
                raise ValueError(f"mode {m}: rank {r} exceeds extent {d}")
    except ValueError as exc:
        raise UsageError(str(exc))
    entries = int(np.prod(dims, dtype=object))
    if full_output and entries > FULL_OUTPUT_CAP and not force:
        raise UsageError(f"--full-output would materialize {entries} entries "
                         f"(cap {FULL_OUTPUT_CAP}); pass --force to override")
    try:
        x = read_tensor_device(input_path, dtype=dtype or torch.float64)
    except (TensorFormatError, OSError) as exc:
        print(f"error: {exc}", file=err)
        return DATA_ERROR

    t0 = time.perf_counter()
    res = rtcur(x, cfg)
    wall = time.perf_counter() - t0

    os.makedirs(out_dir, exist_ok=True)
    outputs = []

    def emit(name, writer):
        writer(os.path.join(out_dir, name))
        outputs.append(name)

    emit("core.tnsr", lambda p: write_tensor(p, res.cur.core))
    for m, fib in enumerate(res.cur.fibers, start=1):
        emit(f"fibers_mode{m}.tnsr", lambda p, v=fib: _write_matrix(p, v))
    for m, fac in enumerate(res.cur.factors, start=1):
        emit(f"factor_mode{m}.tnsr", lambda p, v=fac: _write_matrix(p, v))
    emit("sparse_core.tnsr", lambda p: write_tensor(p, DenseTensor._wrap(np.asfortranarray(res.sparse.core))))
    for m, blk in enumerate(res.sparse.fibers, start=1):
        emit(f"sparse_fibers_mode{m}.tnsr", lambda p, v=blk: _write_matrix(p, v))

    idx = res.sparse.indices
    with open(os.path.join(out_dir, "indices.json"), "w") as f:
        json.dump({"rows": [r.tolist() for r in idx.rows], "cols": [c.tolist() for c in idx.cols]}, f)
    outputs.append("indices.json")
    with open(os.path.join(out_dir, "error_history.csv"), "w") as f:
        f.write("iteration,e\n")
        for k, e in enumerate(res.error_history, start=1):
            f.write(f"{k},{e!r}\n")
    outputs.append("error_history.csv")

    if full_output:
        from .full import full_output as _full

        L, S, _ = _full(res)
        emit("L.tnsr", lambda p: write_tensor_device(p, L))
        emit("S.tnsr", lambda p: write_tensor_device(p, S))

    rows, cols = cfg.resolve_sample_sizes(x.shape)
    _write_manifest(os.path.join(out_dir, "manifest.txt"), [
        ("command", "solve"),
        ("input", input_path),
        ("input_sha256", _sha256(input_path)),
        ("dims", tuple(x.shape)),
        ("ranks", cfg.ranks),
        ("eps", cfg.eps),
        ("zeta0", "inf-norm" if cfg.zeta0 is None else cfg.zeta0),
        ("gamma", cfg.gamma),
        ("upsilon", cfg.upsilon),
        ("variant", cfg.variant),
        ("max_iters", cfg.max_iters),
        ("seed", cfg.seed),
        ("row_samples", rows),
        ("col_samples", cols),
        ("backend", "b200"),
        ("iterations", res.iterations),
        ("converged", res.converged),
        ("final_error", res.error_history[-1]),
        ("zeta_final", res.zeta_final),
        ("resamples", res.iterations - 1 if cfg.variant == "R" else 0),
        ("outputs", ",".join(outputs)),
        ("wall_seconds", wall),
    ])
    return 0 if res.converged else NO_CONVERGENCE
