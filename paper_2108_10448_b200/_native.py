"""ctypes binding of librtcur_b200.so (include/rtcur_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every entry point raises.  Status codes map to the
reference's exception types (solver.py / fiber_cur.py / linalg.py raise
ValueError, IndexError, ArithmeticError).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# (RTCUR_LIB: another build of the same library, for A/B runs of compile-time variants)
LIB_PATH = os.environ.get("RTCUR_LIB") or os.path.join(_HERE, "_lib", "librtcur_b200.so")

(RTCUR_OK, RTCUR_E_VALUE, RTCUR_E_INDEX, RTCUR_E_ARITH, RTCUR_E_CUDA, RTCUR_E_UNSUPPORTED, RTCUR_E_FORMAT,
 RTCUR_E_NOTFOUND, RTCUR_E_IO) = range(9)
RTCUR_F64, RTCUR_F32 = 0, 1

# every symbol include/rtcur_b200.h declares
EXPORTED = (
    "rtcur_last_error", "rtcur_version", "rtcur_launch_count", "rtcur_gather_columns", "rtcur_hard_threshold",
    "rtcur_truncated_svd", "rtcur_engine_plan", "rtcur_engine_create", "rtcur_engine_destroy", "rtcur_engine_bind",
    "rtcur_engine_absmax", "rtcur_engine_set_sample", "rtcur_engine_gather", "rtcur_engine_xblocks_offset", "rtcur_engine_iterate",
    "rtcur_engine_iterate_async", "rtcur_engine_iterate_wait", "rtcur_engine_set_eps", "rtcur_engine_reset", "rtcur_engine_can_speculate",
    "rtcur_engine_last_stop", "rtcur_engine_iterate_cancel",
    "rtcur_engine_export_blocks", "rtcur_engine_export_cur", "rtcur_engine_full_output",
    "rtcur_engine_full_scratch_bytes", "rtcur_engine_profile", "rtcur_engine_profile_phases", "rtcur_engine_set_graphs", "rtcur_engine_absmax_begin", "rtcur_engine_absmax_end", "rtcur_engine_profile_read",
    "rtcur_append_distinct", "rtcur_generate_tucker", "rtcur_tnsr_read_header", "rtcur_tnsr_load", "rtcur_tnsr_store",
    "rtcur_scatter_outliers", "rtcur_abs_sum", "rtcur_ap_threshold", "rtcur_ap_residual", "rtcur_abs_max", "rtcur_engine_bind_mode_copies", "rtcur_engine_build_mode_copy",
    "rtcur_transpose_mode", "rtcur_engine_set_shards", "rtcur_engine_shard_plan", "rtcur_engine_shard_pack",
    "rtcur_engine_shard_unpack", "rtcur_draw_distinct",
)
PHASES = ("absmax", "prep", "gather", "threshold", "gram", "eig", "svdpost", "apass", "gpass", "wcols", "error",
          "export", "full")

_lib = None

c_i64 = ctypes.c_int64
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_dp = ctypes.POINTER(ctypes.c_double)
c_vp = ctypes.c_void_p


class NativeUnavailable(RuntimeError):
    pass


def _keep_large_host_blocks():
    """Results are returned as fresh host arrays (tens to hundreds of MB).  glibc
    serves blocks above its mmap threshold (<= 32 MB) with fresh mappings, so every
    solve's export page-faults its destination pages again (measured: 4 -> 31 ms for
    config 1's 64 MB of blocks).  Keep such blocks on the heap so freed result
    memory is reused without faults.  RTCUR_NO_MALLOPT=1 leaves malloc alone."""
    if os.environ.get("RTCUR_NO_MALLOPT") == "1":
        return
    try:
        libc = ctypes.CDLL("libc.so.6")
        M_TRIM_THRESHOLD, M_MMAP_THRESHOLD = -1, -3
        libc.mallopt(M_MMAP_THRESHOLD, 1 << 30)
        libc.mallopt(M_TRIM_THRESHOLD, 1 << 31 - 1)
    except (OSError, AttributeError):
        pass


def load(path: str = LIB_PATH):
    """Load the sm_100a library (no fallback: raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    _keep_large_host_blocks()
    lib.rtcur_last_error.restype = ctypes.c_char_p
    lib.rtcur_version.restype = ctypes.c_char_p
    lib.rtcur_launch_count.restype = ctypes.c_ulonglong
    lib.rtcur_gather_columns.argtypes = [c_vp, ctypes.c_int, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]
    lib.rtcur_hard_threshold.argtypes = [c_vp, c_i64, ctypes.c_double, c_vp, c_vp]
    lib.rtcur_truncated_svd.argtypes = [c_vp, c_i64, c_i64, ctypes.c_int, c_vp, c_vp, c_vp, c_vp]
    lib.rtcur_engine_plan.argtypes = [ctypes.c_int, c_i64p, c_i32p, c_i64p, c_i64p, ctypes.c_int, c_i64p, c_i64p,
                                      c_i64p]
    lib.rtcur_engine_create.argtypes = [ctypes.POINTER(c_vp), ctypes.c_int, c_i64p, c_i32p, c_i64p, c_i64p,
                                        ctypes.c_int, c_vp, c_i64, c_i64, c_i64, c_vp]
    lib.rtcur_engine_destroy.argtypes = [c_vp]
    lib.rtcur_engine_bind.argtypes = [c_vp, c_vp]
    lib.rtcur_engine_absmax.argtypes = [c_vp, c_dp]
    lib.rtcur_engine_set_sample.argtypes = [c_vp, ctypes.POINTER(c_i64p), ctypes.POINTER(c_i64p)]
    lib.rtcur_engine_gather.argtypes = [c_vp]
    lib.rtcur_draw_distinct.restype = c_i64
    lib.rtcur_draw_distinct.argtypes = [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64]
    lib.rtcur_engine_set_shards.argtypes = [c_vp, ctypes.c_int, ctypes.c_int, c_i64p]
    lib.rtcur_engine_shard_plan.argtypes = [c_vp, c_i64p]
    lib.rtcur_engine_shard_pack.argtypes = [c_vp, c_vp]
    lib.rtcur_engine_shard_unpack.argtypes = [c_vp, c_vp, c_i64]
    lib.rtcur_engine_xblocks_offset.argtypes = [c_vp, c_i64p]
    lib.rtcur_engine_iterate.argtypes = [c_vp, ctypes.c_double, ctypes.c_int, c_dp, c_i32p]
    lib.rtcur_engine_iterate_async.argtypes = [c_vp, ctypes.c_double, ctypes.c_int]
    lib.rtcur_engine_iterate_wait.argtypes = [c_vp, c_dp, c_i32p]
    lib.rtcur_engine_set_eps.argtypes = [c_vp, ctypes.c_double]
    lib.rtcur_engine_reset.argtypes = [c_vp]
    lib.rtcur_engine_build_mode_copy.argtypes = [c_vp, ctypes.c_int, c_vp]
    lib.rtcur_engine_can_speculate.argtypes = [c_vp]
    lib.rtcur_engine_last_stop.argtypes = [c_vp]
    lib.rtcur_engine_iterate_cancel.argtypes = [c_vp]
    lib.rtcur_engine_export_blocks.argtypes = [c_vp, c_vp, c_vp, c_vp]
    lib.rtcur_engine_export_cur.argtypes = [c_vp, ctypes.POINTER(c_dp), ctypes.POINTER(c_dp), ctypes.POINTER(c_dp),
                                            ctypes.POINTER(c_dp), c_dp]
    lib.rtcur_engine_full_output.argtypes = [c_vp, ctypes.c_double, c_vp, c_vp, c_vp, c_dp]
    lib.rtcur_engine_full_scratch_bytes.argtypes = [c_vp]
    lib.rtcur_engine_full_scratch_bytes.restype = c_i64
    lib.rtcur_engine_profile.argtypes = [c_vp, ctypes.c_int]
    lib.rtcur_engine_profile_phases.argtypes = [c_vp, ctypes.c_uint32]
    lib.rtcur_engine_set_graphs.argtypes = [c_vp, ctypes.c_int]
    lib.rtcur_engine_absmax_begin.argtypes = [c_vp]
    lib.rtcur_engine_absmax_end.argtypes = [c_vp, c_dp]
    lib.rtcur_engine_profile_read.argtypes = [c_vp, c_dp, c_i64p, ctypes.c_int, ctypes.c_int]
    lib.rtcur_append_distinct.argtypes = [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64]
    lib.rtcur_append_distinct.restype = c_i64
    lib.rtcur_generate_tucker.argtypes = [c_vp, c_vp, c_i64, ctypes.c_int, c_i64, c_i64, c_i64, ctypes.c_int,
                                          ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_int, c_vp, c_vp,
                                          c_dp, c_vp]
    lib.rtcur_scatter_outliers.argtypes = [c_vp, c_vp, c_vp, c_i64, ctypes.c_double, c_vp, c_vp]
    lib.rtcur_abs_sum.argtypes = [c_vp, c_i64, c_vp, c_dp, c_vp]
    lib.rtcur_ap_threshold.argtypes = [c_vp, c_vp, c_i64, ctypes.c_double, c_vp, c_vp, c_vp]
    lib.rtcur_ap_residual.argtypes = [c_vp, c_vp, c_vp, c_i64, c_vp, c_dp, c_vp]
    lib.rtcur_abs_max.argtypes = [c_vp, ctypes.c_int, c_i64, c_vp, c_dp, c_vp]
    lib.rtcur_engine_bind_mode_copies.argtypes = [c_vp, ctypes.POINTER(c_vp)]
    lib.rtcur_transpose_mode.argtypes = [c_vp, ctypes.c_int, ctypes.c_int, c_i64p, ctypes.c_int, c_vp, c_vp]
    lib.rtcur_tnsr_read_header.argtypes = [ctypes.c_char_p, ctypes.c_int, c_i32p, c_i32p, c_i64p, ctypes.c_int, c_i64p]
    lib.rtcur_tnsr_load.argtypes = [ctypes.c_char_p, c_i64, c_i64, ctypes.c_int, c_vp, c_vp]
    lib.rtcur_tnsr_store.argtypes = [ctypes.c_char_p, ctypes.c_int, c_i64p, ctypes.c_int, c_vp, c_vp]
    for name in EXPORTED:
        if not hasattr(lib, name):
            raise NativeUnavailable(f"{path} does not export {name}")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == RTCUR_OK:
        return
    msg = (_lib.rtcur_last_error() or b"").decode()
    if status == RTCUR_E_VALUE:
        raise ValueError(msg)
    if status == RTCUR_E_INDEX:
        raise IndexError(msg)
    if status == RTCUR_E_ARITH:
        raise ArithmeticError(msg)
    if status == RTCUR_E_FORMAT:
        from .tensorfile import TensorFormatError

        raise TensorFormatError(msg)
    if status == RTCUR_E_NOTFOUND:
        raise FileNotFoundError(msg)
    if status == RTCUR_E_IO:
        raise OSError(msg)
    raise RuntimeError(f"rtcur_b200 status {status}: {msg}")


def launch_count() -> int:
    return int(load().rtcur_launch_count())


def i64_array(values):
    arr = (ctypes.c_int64 * len(values))(*[int(v) for v in values])
    return arr


def i32_array(values):
    return (ctypes.c_int32 * len(values))(*[int(v) for v in values])
