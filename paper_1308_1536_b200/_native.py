"""ctypes binding of libdetseries_b200.so (the C ABI of include/detseries_b200.h).

The library is built in-tree (paper_1308_1536_b200/libdetseries_b200.so, see
__graft_entry__.build()).  There is no CPU fallback: when the library or a CUDA
device is missing, `lib()` raises DeviceUnavailable.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceUnavailable
from .soa import ds_soa

LIB_NAME = "libdetseries_b200.so"
LIB_PATH = os.environ.get("DS_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

DS_OK, DS_ZERO_PIVOT, DS_PRECISION_MISMATCH, DS_INVALID = 0, 1, 2, 3
DS_CUDA, DS_NCCL, DS_OOM, DS_OVERFLOW = 4, 5, 6, 7
DS_KIND_REAL, DS_KIND_COMPLEX = 0, 1

# every symbol include/detseries_b200.h declares (checked by the CPU tests)
EXPORTS = ("ds_version", "ds_create", "ds_destroy", "ds_load", "ds_fetch", "ds_run", "ds_pivot_buffer",
           "ds_pivot_stage", "ds_step", "ds_status", "ds_results_fetch", "ds_set_det", "ds_stream",
           "ds_launch_count", "ds_last_error", "ds_scalar_op", "ds_set_stream", "ds_use_pivot_buffer",
           "ds_pivot_copy", "ds_snapshot", "ds_profile", "ds_profile_read", "ds_counters", "ds_lookahead_enable", "ds_lookahead_stream",
           "ds_lookahead_pivot", "ds_lookahead_mult", "ds_set_pivot_mode", "ds_swaps_fetch",
           "ds_results_fetch_range", "ds_generate", "ds_stream_minors", "ds_stream_flush",
           "ds_update_rows", "ds_create_block", "ds_pivot_load")


class ds_results(ctypes.Structure):
    _fields_ = [("pivots", ds_soa), ("dets", ds_soa), ("signed_minors", ds_soa), ("normalized", ds_soa),
                ("row_flags", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no device access)."""
    if not os.path.exists(path):
        raise DeviceUnavailable(f"{path} is missing: build it with __graft_entry__.build() "
                                f"(make -C paper_1308_1536_b200/csrc); there is no CPU fallback")
    L = ctypes.CDLL(path)
    P, I, L64, VP = ctypes.POINTER, ctypes.c_int, ctypes.c_long, ctypes.c_void_p
    S = P(ds_soa)
    sig = {
        "ds_version": (ctypes.c_char_p, []),
        "ds_create": (I, [P(VP), I, L64, I, I, I, I]),
        "ds_destroy": (None, [VP]),
        "ds_load": (I, [VP, S]),
        "ds_fetch": (I, [VP, S]),
        "ds_run": (I, [VP, I, I, I, I, P(ds_results), P(I)]),
        "ds_pivot_buffer": (I, [VP, P(VP), P(ctypes.c_size_t)]),
        "ds_pivot_stage": (I, [VP, I]),
        "ds_step": (I, [VP, I, I, I]),
        "ds_status": (I, [VP, P(I)]),
        "ds_results_fetch": (I, [VP, I, P(ds_results)]),
        "ds_results_fetch_range": (I, [VP, I, I, I, I, P(ds_results)]),
        "ds_generate": (I, [VP, I, ctypes.c_uint64]),
        "ds_stream_minors": (I, [VP, I, VP, VP]),
        "ds_stream_flush": (I, [VP, I, I]),
        "ds_update_rows": (I, [VP, P(ds_soa)]),
        "ds_create_block": (I, [P(VP), I, ctypes.c_long, I, I, I, I]),
        "ds_pivot_load": (I, [VP, I, P(ds_soa)]),
        "ds_set_det": (I, [VP, S]),
        "ds_stream": (VP, [VP]),
        "ds_launch_count": (ctypes.c_int64, [VP]),
        "ds_last_error": (ctypes.c_char_p, [VP]),
        "ds_scalar_op": (I, [I, I, L64, I, S, S, S]),
        "ds_set_stream": (I, [VP, VP]),
        "ds_use_pivot_buffer": (I, [VP, VP, ctypes.c_size_t]),
        "ds_pivot_copy": (I, [VP, VP]),
        "ds_snapshot": (I, [VP, I]),
        "ds_profile": (I, [VP, I]),
        "ds_profile_read": (I, [VP, P(ctypes.c_double), P(ctypes.c_int64), P(ctypes.c_double)]),
        "ds_counters": (I, [VP, P(ctypes.c_int64), ctypes.c_int]),
        "ds_lookahead_enable": (I, [VP, I]),
        "ds_lookahead_stream": (I, [VP, P(VP)]),
        "ds_lookahead_pivot": (I, [VP, I, VP]),
        "ds_lookahead_mult": (I, [VP, I, VP]),
        "ds_set_pivot_mode": (I, [VP, I]),
        "ds_swaps_fetch": (I, [VP, I, P(ctypes.c_uint8)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


def lib():
    """The loaded library; raises DeviceUnavailable without a CUDA device."""
    global _lib
    with _lock:
        if _lib is None:
            _lib = load_library()
    if not _cuda_available():
        raise DeviceUnavailable("no CUDA device visible: the elimination runs only on the GPU "
                                "(no CPU fallback)")
    return _lib


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def last_error(ctx=None) -> str:
    if _lib is None:
        return ""
    s = _lib.ds_last_error(ctx)
    return s.decode(errors="replace") if s else ""
