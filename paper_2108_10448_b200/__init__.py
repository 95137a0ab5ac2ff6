"""paper_2108_10448_b200 -- B200-native RTCUR (Robust Tensor CUR, arXiv 2108.10448).

Drop-in for the reference package's solver entry point
(/root/reference/pkg/src/rtcur/solver.py:260 ``rtcur(x, cfg, record_trace)``):
same ``SolverConfig`` / ``SolveResult`` / ``FiberCur`` surface, RTCUR-F and
RTCUR-R, with the per-iteration fiber-CUR alternating-projection loop run by
hand-written sm_100a CUDA kernels (librtcur_b200.so, C ABI in
include/rtcur_b200.h).
"""

from .fiber_cur import FiberCur, SampleIndices, TruncatedSvd, draw_sample_indices, sample_indices, sample_sizes
from .full import cur_reconstruct_full, full_output
from .solver import (DenseTensorAccessor, SolveResult, SolverConfig, SparseEstimate, TensorAccessor,
                     hard_threshold, rtcur, sampled_relative_error, zeta_schedule)
from .tensor import DenseTensor, DeviceTensor
from .tensorfile import (TensorFormatError, read_header, read_tensor, read_tensor_device, write_tensor,
                         write_tensor_device)

__all__ = [
    "rtcur", "SolverConfig", "SolveResult", "SparseEstimate", "TensorAccessor", "DenseTensorAccessor",
    "hard_threshold", "zeta_schedule", "sampled_relative_error", "FiberCur", "SampleIndices", "TruncatedSvd",
    "sample_sizes", "sample_indices", "draw_sample_indices", "DenseTensor", "DeviceTensor", "full_output",
    "cur_reconstruct_full", "TensorFormatError", "read_header", "read_tensor", "write_tensor", "read_tensor_device",
    "write_tensor_device",
]
