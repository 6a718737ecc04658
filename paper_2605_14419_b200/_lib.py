"""ctypes binding of libzsort_b200.so (the C ABI in include/zsort_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of the sort entry point raises, loudly.
"""

from __future__ import annotations

import ctypes
import os

from . import build as _build

_lib = None

I64 = ctypes.c_int64
I32 = ctypes.c_int32
P = ctypes.c_void_p
SZ = ctypes.c_size_t


class ZsbConfig(ctypes.Structure):
    _fields_ = [
        ("alpha", ctypes.c_double),
        ("insertion_threshold", I64),
        ("counting_range_threshold", I64),
        ("depth_guard", I64),
        ("collect_stats", I32),
        ("mapping", I32),
    ]


ZSB_OK, ZSB_ERR_ARG, ZSB_ERR_DTYPE, ZSB_ERR_NAN, ZSB_ERR_WORKSPACE, ZSB_ERR_CUDA = range(6)

# Every symbol declared in include/zsort_b200.h (checked by tests/test_abi.py).
EXPORTS = (
    "zsb_workspace_bytes", "zsb_sort", "zsb_rec_workspace_bytes", "zsb_sort_rec", "zsb_moments", "zsb_histogram", "zsb_scatter",
    "zsb_check_workspace_bytes", "zsb_check_sorted", "zsb_last_error", "zsb_version",
    "zsb_timing_enable", "zsb_timing_read", "zsb_timing_records",
    "zsb_local_moments", "zsb_bucket_histogram", "zsb_bucket_minmax", "zsb_partition_workspace_bytes",
    "zsb_partition_to_ranks", "zsb_range_histogram", "zsb_occurrence_workspace_bytes", "zsb_occurrence_index",
    "zsb_generate", "zsb_check_violations", "zsb_partition_send",
)

PHASES = ("moments", "histogram", "scan", "scatter", "classify", "finish", "recursion_stats", "misc")


def load(auto_build: bool = True):
    """Load (building in-tree first if sources are newer) the C-ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    variant = os.environ.get("ZSB_LIB_VARIANT")  # experiments: an in-tree build variant, libzsort_b200_<v>.so
    if variant:
        path, auto_build = path[:-3] + f"_{variant}.so", False
    if auto_build and _build.needs_build():
        try:
            _build.build()
        except Exception as exc:  # no nvcc on this host: use what was shipped
            if not os.path.exists(path):
                raise RuntimeError(f"libzsort_b200.so is missing and cannot be built: {exc}") from exc
    if not os.path.exists(path):
        raise RuntimeError(f"libzsort_b200.so not found at {path}; run python -m paper_2605_14419_b200.build")
    L = ctypes.CDLL(path)
    L.zsb_workspace_bytes.argtypes = [I64, I32, I32, ctypes.POINTER(ZsbConfig)]
    L.zsb_workspace_bytes.restype = SZ
    L.zsb_sort.argtypes = [P, I32, P, I32, P, P, I64, ctypes.POINTER(ZsbConfig), P, SZ, P, P]
    L.zsb_sort.restype = ctypes.c_int
    L.zsb_rec_workspace_bytes.argtypes = [I64, I32, I32, I64]
    L.zsb_rec_workspace_bytes.restype = SZ
    L.zsb_sort_rec.argtypes = [P, I32, P, I32, P, P, I64, I64, ctypes.c_double, ctypes.c_double, I64,
                               ctypes.POINTER(ZsbConfig), P, SZ, P, P]
    L.zsb_sort_rec.restype = ctypes.c_int
    L.zsb_moments.argtypes = [P, I32, I64, P, SZ, P, P, P, P]
    L.zsb_moments.restype = ctypes.c_int
    L.zsb_histogram.argtypes = [P, I32, I64, P, I64, P, P, SZ, P]
    L.zsb_histogram.restype = ctypes.c_int
    L.zsb_scatter.argtypes = [P, I32, P, I32, I64, P, I64, P, P, P, SZ, P]
    L.zsb_scatter.restype = ctypes.c_int
    L.zsb_check_workspace_bytes.argtypes = [I64]
    L.zsb_check_workspace_bytes.restype = SZ
    L.zsb_check_sorted.argtypes = [P, P, P, I32, I32, I64, I64, P, P, P]
    L.zsb_check_sorted.restype = ctypes.c_int
    D = ctypes.c_double
    L.zsb_local_moments.argtypes = [P, I32, I64, D, P, P, P]
    L.zsb_local_moments.restype = ctypes.c_int
    L.zsb_occurrence_workspace_bytes.argtypes = []
    L.zsb_occurrence_workspace_bytes.restype = SZ
    L.zsb_occurrence_index.argtypes = [P, I32, I64, ctypes.c_uint64, I64, P, P, P]
    L.zsb_occurrence_index.restype = ctypes.c_int
    L.zsb_generate.argtypes = [I32, I64, I64, I64, ctypes.c_uint64, P, P, P]
    L.zsb_generate.restype = ctypes.c_int
    L.zsb_partition_send.argtypes = [P, I32, P, I32, I64, I32, P, P, P, P, SZ, P]
    L.zsb_partition_send.restype = ctypes.c_int
    L.zsb_check_violations.argtypes = [I32]
    L.zsb_check_violations.restype = I64
    L.zsb_bucket_histogram.argtypes = [P, I32, I64, P, I64, P, P]
    L.zsb_bucket_histogram.restype = ctypes.c_int
    L.zsb_bucket_minmax.argtypes = [P, I32, I64, P, I64, I32, P, P, P, P]
    L.zsb_bucket_minmax.restype = ctypes.c_int
    L.zsb_range_histogram.argtypes = [P, I32, I64, P, I64, I32, P, P, P, P, I32, P, P]
    L.zsb_range_histogram.restype = ctypes.c_int
    L.zsb_partition_workspace_bytes.argtypes = [I64, I32, I32]
    L.zsb_partition_workspace_bytes.restype = SZ
    L.zsb_partition_to_ranks.argtypes = [P, I32, P, I32, I64, P, I64, I64, I32, P, P, P, P, P, P, P, SZ, P]
    L.zsb_partition_to_ranks.restype = ctypes.c_int
    L.zsb_timing_enable.argtypes = [I32]
    L.zsb_timing_enable.restype = None
    L.zsb_timing_read.argtypes = [P, P, I32, I32]
    L.zsb_timing_read.restype = I32
    L.zsb_timing_records.argtypes = [P, I32]
    L.zsb_timing_records.restype = I32
    L.zsb_last_error.argtypes = []
    L.zsb_last_error.restype = ctypes.c_char_p
    L.zsb_version.argtypes = []
    L.zsb_version.restype = ctypes.c_char_p
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a ZSB_ERR_* code to the reference's exception types."""
    if rc == ZSB_OK:
        return
    msg = (_lib.zsb_last_error() or b"").decode()
    if rc in (ZSB_ERR_ARG, ZSB_ERR_NAN):
        raise ValueError(msg)
    if rc == ZSB_ERR_DTYPE:
        raise TypeError(msg)
    raise RuntimeError(f"zsort_b200 error {rc}: {msg}")
