"""TNSR v1 tensor files (mirror of /root/reference/pkg/src/rtcur/tensorfile.py).

Layout, all little-endian: "TNSR" | u16 version (1) | u16 mode count n |
n u64 extents | prod(extents) IEEE-754 doubles, mode-1 fastest.

Host API (same names, semantics and error texts as the reference):
``read_header``, ``read_tensor`` (-> DenseTensor), ``write_tensor``.
Device API (the B200 path): ``read_tensor_device`` streams
the payload from disk straight into HBM through pinned double buffers
(pread threads overlapped with async H2D; optional fp32 rounding and mode-1
slab extraction for sharded runs), ``write_tensor_device`` streams a
DeviceTensor back to a file (D2H of the next chunk overlapped with the write
of the current one).  Header validation runs in the native library
(``rtcur_tnsr_read_header``) for both, so every TensorFormatError names the
offending byte offset exactly as the reference does (tensorfile.py:50-115).
"""

from __future__ import annotations

import ctypes
import math
import os
import struct

import numpy as np

from . import _native as nat
from .tensor import DenseTensor, DeviceTensor, as_shape

__all__ = ["MAGIC", "FORMAT_VERSION", "TensorFormatError", "read_header", "read_tensor", "write_tensor",
           "read_tensor_device", "write_tensor_device"]

MAGIC = b"TNSR"
FORMAT_VERSION = 1
_MAX_MODES = 65535


class TensorFormatError(ValueError):
    """Malformed tensor file; the message names the offending byte offset."""


def _header(path, check_payload: bool):
    lib = nat.load()
    ver = ctypes.c_int32()
    n = ctypes.c_int32()
    dims = (ctypes.c_int64 * 64)()
    off = ctypes.c_int64()
    nat.check(lib.rtcur_tnsr_read_header(os.fsencode(os.fspath(path)), int(bool(check_payload)), ctypes.byref(ver),
                                         ctypes.byref(n), dims, 64, ctypes.byref(off)))
    if n.value > 64:   # rare: re-read with room for every extent
        dims = (ctypes.c_int64 * n.value)()
        nat.check(lib.rtcur_tnsr_read_header(os.fsencode(os.fspath(path)), int(bool(check_payload)),
                                             ctypes.byref(ver), ctypes.byref(n), dims, n.value, ctypes.byref(off)))
    return int(ver.value), tuple(int(dims[m]) for m in range(n.value)), int(off.value)


def read_header(path) -> tuple[int, tuple[int, ...]]:
    """Format version and extents, without touching the payload (tensorfile.py:87-92)."""
    version, dims, _ = _header(path, False)
    return version, dims


def read_tensor(path) -> DenseTensor:
    """Host DenseTensor (tensorfile.py:94-115): validated header, exact payload size."""
    _, dims, off = _header(path, True)
    count = math.prod(dims)
    with open(path, "rb") as f:
        f.seek(off)
        flat = np.fromfile(f, dtype="<f8", count=count)
    if flat.size != count:   # racing truncation after the header check
        raise TensorFormatError(f"{path}: payload at byte {off} holds {flat.size * 8} bytes, "
                                f"dims {dims} require {count * 8}")
    return DenseTensor._wrap(np.reshape(flat.astype(np.float64, copy=False), dims, order="F"))


def write_tensor(path, t) -> None:
    """tensorfile.py:42-48 for a host DenseTensor; DeviceTensors go through write_tensor_device."""
    if isinstance(t, DeviceTensor):
        write_tensor_device(path, t)
        return
    dims = t.shape
    header = MAGIC + struct.pack("<HH", FORMAT_VERSION, len(dims)) + struct.pack(f"<{len(dims)}Q", *dims)
    payload = t.data.astype("<f8", copy=False)
    with open(path, "wb") as f:
        f.write(header)
        payload.tofile(f)


def read_tensor_device(path, dtype=None, slab=None, stream=None) -> DeviceTensor:
    """Stream a TNSR file into HBM.  dtype: torch.float64 (default) or torch.float32
    (rounded on the device); slab=(lo, hi): only mode-1 rows [lo, hi) (0-based),
    returned as a mode-1-fastest (hi-lo, d_2, ...) tensor."""
    import torch

    _, dims, _ = _header(path, True)
    dtype = dtype or torch.float64
    if dtype not in (torch.float64, torch.float32):
        raise ValueError(f"dtype must be torch.float64 or torch.float32, got {dtype}")
    lo, hi = slab if slab is not None else (0, dims[0])
    if not (0 <= lo < hi <= dims[0]):
        raise ValueError(f"slab {slab} outside mode 1 of extent {dims[0]}")
    shape = (hi - lo,) + tuple(dims[1:])
    dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(math.prod(shape), dtype=dtype, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    nat.check(nat.load().rtcur_tnsr_load(os.fsencode(os.fspath(path)), int(lo), int(hi),
                                         0 if dtype == torch.float64 else 1, out.data_ptr(), st))
    return DeviceTensor(out, shape)


def write_tensor_device(path, t: DeviceTensor, stream=None) -> None:
    """Stream a DeviceTensor (fp64, or fp32 widened exactly) to a TNSR file."""
    import torch

    if not isinstance(t, DeviceTensor):
        raise TypeError("write_tensor_device needs a DeviceTensor")
    shape = as_shape(t.shape)
    if len(shape) > _MAX_MODES:
        raise ValueError(f"{len(shape)} modes exceed the format's u16 mode count")
    dims = (ctypes.c_int64 * len(shape))(*shape)
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    flat = t.flat.contiguous()
    nat.check(nat.load().rtcur_tnsr_store(os.fsencode(os.fspath(path)), len(shape), dims,
                                          0 if flat.dtype == torch.float64 else 1, flat.data_ptr(), st))
