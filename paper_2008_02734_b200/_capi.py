"""ctypes binding of liblmdtw_b200.so (the C ABI in include/lmdtw_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute call raises.  ctypes releases the GIL for the duration
of each foreign call.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LMDTW_LIB_PATH") or os.path.join(_HERE, "liblmdtw_b200.so")

OK, EINVAL, ENOMEM, ECUDA, EINTERNAL = 0, -1, -2, -3, -4
MEM_HOST, MEM_DEVICE = 0, 1

PROGRESS_FN = C.CFUNCTYPE(None, C.c_int64, C.c_int64, C.c_void_p)


class Config(C.Structure):
    _fields_ = [("min_dim", C.c_int32), ("precision", C.c_int32), ("tie", C.c_int32 * 3),
                ("pivot_highest", C.c_int32), ("reserved", C.c_int32 * 4)]


class PivotRec(C.Structure):
    _fields_ = [("i", C.c_int64), ("j", C.c_int64), ("i_off", C.c_int64), ("j_off", C.c_int64),
                ("M", C.c_int64), ("N", C.c_int64), ("sub_i", C.c_int64), ("sub_j", C.c_int64),
                ("diagonal_k", C.c_int64), ("total_at_pivot", C.c_double)]


class AlignInfo(C.Structure):
    _fields_ = [("cost", C.c_double), ("path_len", C.c_int64), ("cells_processed", C.c_int64),
                ("cells_budget", C.c_int64), ("peak_diag_values", C.c_int64),
                ("peak_table_cells", C.c_int64), ("n_pivots", C.c_int64), ("n_levels", C.c_int64),
                ("gpu_launches", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64)]


# Every symbol include/lmdtw_b200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "lmdtw_version", "lmdtw_last_error", "lmdtw_device_count", "lmdtw_max_dim",
    "lmdtw_half_pass", "lmdtw_find_pivot", "lmdtw_dtw_full", "lmdtw_align",
    "lmdtw_align_batch", "lmdtw_result_info", "lmdtw_result_path", "lmdtw_result_pivots",
    "lmdtw_result_free", "lmdtw_path_cost", "lmdtw_diag_length", "lmdtw_cells_upto",
    "lmdtw_peak_retained_values", "lmdtw_launch_count", "lmdtw_pivot_nodes", "lmdtw_leaf_nodes",
    "lmdtw_pivot_combine", "lmdtw_half_pass_shard", "lmdtw_handoff_words", "lmdtw_strip_height",
    "lmdtw_ipc_alloc", "lmdtw_ipc_open", "lmdtw_ipc_close", "lmdtw_ipc_free", "lmdtw_fill_ones",
    "lmdtw_window_dtw", "lmdtw_frame_costs", "lmdtw_path_cost_batch", "lmdtw_discrepancy",
)

_lib = None


def load():
    """Load (never build) the library; raise ImportError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2008_02734_b200/build.py` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.lmdtw_version.restype = C.c_char_p
    L.lmdtw_last_error.restype = C.c_char_p
    L.lmdtw_device_count.restype = C.c_int
    L.lmdtw_max_dim.argtypes = [I32]
    L.lmdtw_max_dim.restype = C.c_int
    L.lmdtw_half_pass.argtypes = [C.c_int, P, I64, P, I64, I32, I64, I32, I32, I32, P, P, P]
    L.lmdtw_half_pass.restype = C.c_int
    L.lmdtw_find_pivot.argtypes = [C.c_int, P, I64, P, I64, I32, I32, I32, I32, P, P, P, P, P, P]
    L.lmdtw_find_pivot.restype = C.c_int
    L.lmdtw_dtw_full.argtypes = [C.c_int, P, I64, P, I64, I32, P, I32, I32, P, P, P, P]
    L.lmdtw_dtw_full.restype = C.c_int
    L.lmdtw_align.argtypes = [C.c_int, P, I64, P, I64, I32, C.POINTER(Config), I32, PROGRESS_FN, P,
                              C.POINTER(P)]
    L.lmdtw_align.restype = C.c_int
    L.lmdtw_align_batch.argtypes = [C.c_int, I32, P, P, P, P, I32, C.POINTER(Config), I32, P]
    L.lmdtw_align_batch.restype = C.c_int
    L.lmdtw_result_info.argtypes = [P, C.POINTER(AlignInfo)]
    L.lmdtw_result_info.restype = C.c_int
    L.lmdtw_result_path.argtypes = [P, P]
    L.lmdtw_result_path.restype = C.c_int
    L.lmdtw_result_pivots.argtypes = [P, P]
    L.lmdtw_result_pivots.restype = C.c_int
    L.lmdtw_result_free.argtypes = [P]
    L.lmdtw_result_free.restype = None
    L.lmdtw_pivot_nodes.argtypes = [C.c_int, P, I64, P, I64, I32, I32, P, I32, I32, I32, P, P]
    L.lmdtw_pivot_nodes.restype = C.c_int
    L.lmdtw_leaf_nodes.argtypes = [C.c_int, P, I64, P, I64, I32, I32, P, P, I32, I32, P, P]
    L.lmdtw_leaf_nodes.restype = C.c_int
    L.lmdtw_pivot_combine.argtypes = [I32, I64, I64, I32, P, P, P, P, P]
    L.lmdtw_half_pass_shard.argtypes = [C.c_int, P, I64, P, I64, I32, I64, I32, I32, I32, I32, I32, P, P, P, P, P]
    L.lmdtw_half_pass_shard.restype = C.c_int
    L.lmdtw_handoff_words.argtypes = [I64, I32]
    L.lmdtw_handoff_words.restype = I64
    L.lmdtw_strip_height.argtypes = [I32, I32]
    L.lmdtw_strip_height.restype = I32
    L.lmdtw_ipc_alloc.argtypes = [C.c_int, I64, P, P]
    L.lmdtw_ipc_open.argtypes = [C.c_int, P, P]
    L.lmdtw_ipc_close.argtypes = [C.c_int, P]
    L.lmdtw_ipc_free.argtypes = [C.c_int, P]
    L.lmdtw_fill_ones.argtypes = [C.c_int, P, I64]
    L.lmdtw_pivot_combine.restype = C.c_int
    L.lmdtw_path_cost.argtypes = [P, I64, P, I64, I32, P, I64, I32, P]
    L.lmdtw_path_cost.restype = C.c_int
    L.lmdtw_window_dtw.argtypes = [C.c_int, P, I64, P, I64, I32, P, P, P, I32, I32, P, P, P, P]
    L.lmdtw_window_dtw.restype = C.c_int
    L.lmdtw_frame_costs.argtypes = [C.c_int, P, P, I64, I32, I32, I32, P]
    L.lmdtw_frame_costs.restype = C.c_int
    L.lmdtw_path_cost_batch.argtypes = [C.c_int, I32, P, P, P, P, I32, P, P, I32, I32, P]
    L.lmdtw_path_cost_batch.restype = C.c_int
    L.lmdtw_discrepancy.argtypes = [C.c_int, P, I64, P, I64, P]
    L.lmdtw_discrepancy.restype = C.c_int
    for f in ("lmdtw_diag_length", "lmdtw_cells_upto", "lmdtw_peak_retained_values"):
        getattr(L, f).argtypes = [I64, I64, I64]
        getattr(L, f).restype = I64
    L.lmdtw_launch_count.restype = I64
    L.lmdtw_profile_enable.argtypes = [C.c_int]
    L.lmdtw_profile_get.argtypes = [P]
    L.lmdtw_stream.argtypes = [C.c_int]
    L.lmdtw_stream.restype = P
    _lib = L
    return L


def check(rc: int):
    """Map a status code to the reference's exception classes."""
    if rc == OK:
        return
    from .core import InvalidInputError
    msg = load().lmdtw_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise InvalidInputError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"liblmdtw_b200: {msg}")


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


_device = int(os.environ.get("LMDTW_DEVICE", "0"))


def set_device(device: int):
    """Select the CUDA device used by subsequent calls from this process."""
    global _device
    _device = int(device)


def get_device() -> int:
    return _device


def launch_count() -> int:
    return int(load().lmdtw_launch_count())


def profile(enable: bool):
    load().lmdtw_profile_enable(1 if enable else 0)


def profile_reset():
    load().lmdtw_profile_reset()


def profile_get() -> dict:
    buf = (C.c_double * 5)()
    load().lmdtw_profile_get(buf)
    return {"wave_ms": buf[0], "wave_launches": int(buf[1]), "wave_cells": int(buf[2]),
            "leaf_ms": buf[3], "leaf_cells": int(buf[4])}


def stream_handle(device: int | None = None) -> int:
    """cudaStream_t (as int) that every kernel of `device` runs on."""
    return int(load().lmdtw_stream(_device if device is None else device) or 0)
