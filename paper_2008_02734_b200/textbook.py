"""Textbook DTW with backpointers: the leaf solver and the "brute-force DTW
with backtrace" entry point (drop-in for the reference's oracle module,
/root/reference/pkg/src/lmdtw/oracle.py; renamed here so it cannot be
confused with this repo's test oracle under oracle/).

The table is filled on the GPU by the strip-wavefront kernel in leaf mode with
2-bit backpointers and walked back on the device.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from .core import (AlignmentResult, InvalidInputError, as_series, check_cost_kind,
                   precision_bits, precision_dtype)

# Backpointer codes; SELF marks the (0, 0) corner (oracle.py:23).
LEFT, UP, DIAG, SELF = 0, 1, 2, 3

#: Default move precedence on ties: diagonal beats left beats up (oracle.py:26).
TIE_DIAG_FIRST = ("diag", "left", "up")
#: Alternate rule: left beats diagonal (oracle.py:28).
TIE_LEFT_FIRST = ("left", "diag", "up")

_MOVE_CODES = {"left": LEFT, "up": UP, "diag": DIAG}


def tie_codes(tie_rule) -> np.ndarray:
    """("diag", "left", "up") -> int8 codes (oracle.py:33-37)."""
    if sorted(tie_rule) != sorted(_MOVE_CODES):
        raise InvalidInputError(f"tie rule must order {tuple(_MOVE_CODES)}, got {tie_rule!r}")
    return np.array([_MOVE_CODES[m] for m in tie_rule], dtype=np.int8)


def _run(X, Y, tie_rule, precision, want_table):
    X, Y = as_series(X), as_series(Y)
    if X.dim != Y.dim:
        raise InvalidInputError(f"feature dimension mismatch: {X.dim} vs {Y.dim}")
    dtype = precision_dtype(precision)
    tie = tie_codes(tie_rule).astype(np.int32)
    M, N = len(X), len(Y)
    xf = np.ascontiguousarray(X.frames, dtype=np.float32)
    yf = np.ascontiguousarray(Y.frames, dtype=np.float32)
    path = np.empty((M + N - 1, 2), np.int64)
    cost = C.c_double()
    plen = C.c_int64()
    table = None
    if want_table:
        try:
            table = np.empty((M, N), dtype)
        except (MemoryError, ValueError) as e:  # numpy refuses absurd sizes
            raise MemoryError(str(e))
    _capi.check(_capi.load().lmdtw_dtw_full(
        _capi.get_device(), _capi.ptr(xf), M, _capi.ptr(yf), N, X.dim, _capi.ptr(tie),
        precision_bits(precision), _capi.MEM_HOST, C.byref(cost), _capi.ptr(path), C.byref(plen),
        None if table is None else _capi.ptr(table)))
    return float(cost.value), path[:plen.value].copy(), dtype, table, M, N


def dtw_full(X, Y, cost: str = "euclidean", tie_rule=TIE_DIAG_FIRST,
             precision=64) -> AlignmentResult:
    """Exact DTW by filling the full table (oracle.py:105-131).  Raises
    MemoryError when the device cannot hold the 2-bit backpointer grid."""
    check_cost_kind(cost)
    c, path, dtype, _, M, N = _run(X, Y, tie_rule, precision, False)
    return AlignmentResult(
        cost=c, path=path, cells_processed=int(M * N), cells_budget=int(M * N),
        precision=str(dtype), algorithm="dtw", peak_table_cells=int(M * N))


def accumulated_cost_table(X, Y, precision=64) -> np.ndarray:
    """Full D(i, j) table (oracle.py:134-141; test instrumentation)."""
    table = _run(X, Y, TIE_DIAG_FIRST, precision, True)[3]
    return table


def backtrace(P: np.ndarray) -> np.ndarray:
    """Follow uint8 backpointers from the bottom-right corner (oracle.py:85-102).

    Host helper for callers that hold a backpointer grid; the device solver
    walks its own packed grid inside liblmdtw_b200.so.
    """
    M, N = P.shape
    i, j = M - 1, N - 1
    rev = [(i, j)]
    while (i, j) != (0, 0):
        move = P[i, j]
        if move == LEFT:
            j -= 1
        elif move == UP:
            i -= 1
        elif move == DIAG:
            i -= 1
            j -= 1
        else:
            raise RuntimeError(f"backtrace hit SELF at ({i}, {j}) before (0, 0)")
        rev.append((i, j))
    return np.array(rev[::-1], dtype=np.int64)
