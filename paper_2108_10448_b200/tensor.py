"""Host-side tensor containers and index arithmetic (mirror of the reference's
``rtcur.tensor``, /root/reference/pkg/src/rtcur/tensor.py).

Layout contract (tensor.py:1-10): mode 1 varies fastest; element
(i_1, ..., i_n) (1-based) lives at flat offset sum_m (i_m - 1) prod_{l<m} d_l.
A C-contiguous buffer of shape (d_n, ..., d_1) has identical memory, so the
device path adopts the same bytes with no transpose.

``DenseTensor`` is the reference's immutable fp64 host tensor;
``DeviceTensor`` holds the same layout in HBM (torch CUDA storage, fp64 or
fp32) and is what the B200 solver consumes.
"""

from __future__ import annotations

from typing import Iterable, Sequence

import math

import numpy as np

__all__ = ["DenseTensor", "DeviceTensor", "mode_stride", "decode_fiber_columns", "fiber_base_offsets", "as_shape"]


def as_shape(dims: Sequence[int]) -> tuple[int, ...]:
    """tensor.py:35-47."""
    shape = tuple(int(d) for d in dims)
    if len(shape) == 0:
        raise ValueError("shape needs at least one mode")
    total = 1
    for m, d in enumerate(shape, start=1):
        if d < 1:
            raise ValueError(f"mode {m} has nonpositive extent {d}")
        total *= d
        if total >= 2 ** 63:
            raise ValueError(f"element count of shape {shape} is not addressable")
    return shape


def _strides(shape):
    out, acc = [], 1
    for d in shape:
        out.append(acc)
        acc *= d
    return tuple(out)


class DenseTensor:
    """Immutable float64 tensor, mode-1-fastest (tensor.py:66-136)."""

    __slots__ = ("_array",)

    def __init__(self, data: Iterable[float], shape: Sequence[int]):
        shape = as_shape(shape)
        flat = np.asarray(data, dtype=np.float64).reshape(-1)
        total = math.prod(shape)
        if flat.size != total:
            raise ValueError(f"data length {flat.size} does not match shape {shape} (expected {total})")
        arr = np.array(flat, dtype=np.float64, copy=True).reshape(shape, order="F")
        arr.flags.writeable = False
        self._array = arr

    @classmethod
    def _wrap(cls, arr: np.ndarray) -> "DenseTensor":
        t = object.__new__(cls)
        if not (arr.flags.f_contiguous and arr.dtype == np.float64 and arr.ndim >= 1):
            raise ValueError("_wrap needs an F-contiguous float64 array")
        as_shape(arr.shape)
        arr.flags.writeable = False
        t._array = arr
        return t

    @classmethod
    def from_array(cls, arr: np.ndarray) -> "DenseTensor":
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim == 0:
            arr = arr.reshape(1)
        return cls._wrap(np.array(arr, dtype=np.float64, order="F", copy=True))

    @classmethod
    def zeros(cls, shape: Sequence[int]) -> "DenseTensor":
        return cls._wrap(np.zeros(as_shape(shape), order="F"))

    @property
    def shape(self) -> tuple[int, ...]:
        return self._array.shape

    @property
    def ndim(self) -> int:
        return self._array.ndim

    @property
    def size(self) -> int:
        return self._array.size

    @property
    def data(self) -> np.ndarray:
        return self._array.reshape(-1, order="F")

    def to_array(self) -> np.ndarray:
        return self._array

    def value_at(self, idx: Sequence[int]) -> float:
        off = 0
        for m, (i, d, s) in enumerate(zip(idx, self.shape, _strides(self.shape)), start=1):
            if not 1 <= int(i) <= d:
                raise IndexError(f"mode {m}: index {i} outside [1, {d}]")
            off += (int(i) - 1) * s
        return float(self.data[off])

    def __repr__(self) -> str:
        return f"DenseTensor(shape={self.shape})"


class DeviceTensor:
    """A mode-1-fastest tensor resident in HBM (fp64 or fp32).

    ``flat`` is a contiguous 1-d torch CUDA tensor of prod(shape) elements.
    """

    __slots__ = ("flat", "shape")

    def __init__(self, flat, shape: Sequence[int]):
        import torch

        shape = as_shape(shape)
        if not isinstance(flat, torch.Tensor) or not flat.is_cuda:
            raise ValueError("DeviceTensor needs a CUDA torch tensor")
        if flat.dtype not in (torch.float64, torch.float32):
            raise ValueError(f"DeviceTensor dtype must be float64 or float32, got {flat.dtype}")
        flat = flat.reshape(-1)
        if not flat.is_contiguous():
            raise ValueError("DeviceTensor storage must be contiguous")
        if flat.numel() != math.prod(shape):
            raise ValueError(f"{flat.numel()} elements do not match shape {shape}")
        self.flat = flat
        self.shape = shape

    @classmethod
    def from_host(cls, x, dtype=None, device=None) -> "DeviceTensor":
        """Upload a DenseTensor (or an F-ordered numpy array) to the GPU."""
        import torch

        if isinstance(x, DenseTensor):
            flat, shape = x.data, x.shape
        else:
            arr = np.asarray(x)
            flat, shape = arr.reshape(-1, order="F"), arr.shape
        t = torch.from_numpy(np.array(flat, copy=True))
        dt = dtype or (torch.float64 if t.dtype == torch.float64 else torch.float32)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        return cls(t.to(device=dev, dtype=dt), shape)

    @classmethod
    def from_torch(cls, t) -> "DeviceTensor":
        """Adopt a torch CUDA tensor of shape (d_1, ..., d_n) laid out mode-1-fastest
        (i.e. ``t.permute(reversed)`` is C-contiguous), without a copy."""
        shape = tuple(t.shape)
        back = t.permute(*reversed(range(t.dim())))
        if not back.is_contiguous():
            raise ValueError("tensor is not mode-1-fastest (F-contiguous)")
        return cls(back.reshape(-1), shape)

    @property
    def dtype(self):
        return self.flat.dtype

    @property
    def size(self) -> int:
        return int(self.flat.numel())

    def to_dense(self) -> DenseTensor:
        return DenseTensor._wrap(
            np.asfortranarray(self.flat.double().cpu().numpy().reshape(self.shape, order="F")))

    def __repr__(self) -> str:
        return f"DeviceTensor(shape={self.shape}, dtype={self.flat.dtype}, device={self.flat.device})"


def mode_stride(shape: Sequence[int], k: int) -> int:
    """tensor.py:243-247."""
    shape = as_shape(shape)
    if not 1 <= k <= len(shape):
        raise ValueError(f"mode {k} out of range for {len(shape)}-mode tensor")
    return _strides(shape)[k - 1]


def decode_fiber_columns(shape: Sequence[int], k: int, cols: np.ndarray) -> tuple[np.ndarray, ...]:
    """tensor.py:250-270."""
    shape = as_shape(shape)
    if not 1 <= k <= len(shape):
        raise ValueError(f"mode {k} out of range for {len(shape)}-mode tensor")
    cols = np.asarray(cols, dtype=np.int64).reshape(-1)
    others = [d for j, d in enumerate(shape, start=1) if j != k]
    total = math.prod(others)
    if cols.size and (cols.min() < 1 or cols.max() > total):
        raise IndexError(f"column index outside [1, {total}] for mode {k} of {shape}")
    rem = cols - 1
    out = []
    for d in others:
        out.append((rem % d) + 1)
        rem = rem // d
    return tuple(out)


def fiber_base_offsets(shape: Sequence[int], k: int, cols: np.ndarray) -> np.ndarray:
    """tensor.py:273-283."""
    shape = as_shape(shape)
    parts = decode_fiber_columns(shape, k, cols)
    st = _strides(shape)
    other = [s for j, s in enumerate(st, start=1) if j != k]
    base = np.zeros(np.asarray(cols).size, dtype=np.int64)
    for idx, s in zip(parts, other):
        base += (idx - 1) * s
    return base
