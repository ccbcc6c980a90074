"""Exact linear-memory DTW by divide and conquer (drop-in for the reference's
divide module, /root/reference/pkg/src/lmdtw/divide.py).

The recursion runs inside liblmdtw_b200.so: one batched launch per recursion
level for all half passes of that level, one for the split-point reduction,
and one batched leaf solve.  Results (path, cost, cells_processed,
peak_diag_values, peak_table_cells, pivot_trace in pre-order DFS) are
identical to the reference's for the same inputs and configuration.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from .core import (AlignmentResult, InvalidInputError, as_series, check_cost_kind,
                   precision_bits, precision_dtype)
from .textbook import TIE_DIAG_FIRST, tie_codes


@dataclass(frozen=True)
class Pivot:
    """A cell on an optimal warping path (divide.py:30-41)."""

    i: int
    j: int
    total_at_pivot: float
    diagonal_k: int


@dataclass(frozen=True)
class LinMdtwConfig:
    """Recursion configuration (divide.py:44-57).  ``parallel_halves`` and
    ``parallel_diagonals`` are accepted for compatibility; the device always
    runs both levels of parallelism and results do not depend on them."""

    min_dim: int = 500
    precision: int = 64
    tie_rule: tuple = TIE_DIAG_FIRST
    pivot_tie_rule: str = "lowest"  # lowest diagonal, then lowest idx
    parallel_halves: bool = False
    parallel_diagonals: bool = False

    def __post_init__(self):
        if self.min_dim < 2:
            raise InvalidInputError("min_dim must be >= 2")
        if self.pivot_tie_rule not in ("lowest", "highest"):
            raise InvalidInputError(f"unknown pivot_tie_rule {self.pivot_tie_rule!r}")


def _c_config(cfg: LinMdtwConfig) -> _capi.Config:
    c = _capi.Config()
    c.min_dim = int(min(cfg.min_dim, 2**31 - 1))
    c.precision = precision_bits(cfg.precision)
    tie = tie_codes(cfg.tie_rule)
    for q in range(3):
        c.tie[q] = int(tie[q])
    c.pivot_highest = 1 if cfg.pivot_tie_rule == "highest" else 0
    return c


def find_pivot(X, Y, cost: str = "euclidean", precision=64, parallel: bool = False,
               pivot_tie_rule: str = "lowest", _inst=None) -> Pivot:
    """Locate a cell on an optimal warping path via half passes from both ends
    (divide.py:97-145): forward to diagonal ceil((M+N-1)/2), reverse to the
    matching diagonal, then argmin of (Df + Db) - Cf over the three shared
    diagonals with the lexicographic tie rule."""
    check_cost_kind(cost)
    X, Y = as_series(X), as_series(Y)
    M, N = len(X), len(Y)
    if M + N - 2 < 2:
        raise InvalidInputError(f"{M}x{N} too small for a pivot search; use dtw_full")
    if X.dim != Y.dim:
        raise InvalidInputError(f"feature dimension mismatch: {X.dim} vs {Y.dim}")
    if pivot_tie_rule not in ("lowest", "highest"):
        raise InvalidInputError(f"unknown pivot_tie_rule {pivot_tie_rule!r}")
    prec = precision_bits(precision)
    xf = np.ascontiguousarray(X.frames, dtype=np.float32)
    yf = np.ascontiguousarray(Y.frames, dtype=np.float32)
    i, j, k, cells, peak = (C.c_int64() for _ in range(5))
    tot = C.c_double()
    _capi.check(_capi.load().lmdtw_find_pivot(
        _capi.get_device(), _capi.ptr(xf), M, _capi.ptr(yf), N, X.dim, prec,
        1 if pivot_tie_rule == "highest" else 0, _capi.MEM_HOST, C.byref(i), C.byref(j),
        C.byref(k), C.byref(tot), C.byref(cells), C.byref(peak)))
    if _inst is not None:
        _inst.add_cells(int(cells.value))
        _inst.saw_diag_run(int(peak.value))
    return Pivot(i=int(i.value), j=int(j.value), total_at_pivot=float(tot.value),
                 diagonal_k=int(k.value))


# PivotRec (include/lmdtw_b200.h) as a numpy record: one .tolist() instead of
# ten ctypes attribute reads per pivot
_PIV_DT = np.dtype([("i", "<i8"), ("j", "<i8"), ("i_off", "<i8"), ("j_off", "<i8"), ("M", "<i8"), ("N", "<i8"),
                    ("sub_i", "<i8"), ("sub_j", "<i8"), ("diagonal_k", "<i8"), ("total_at_pivot", "<f8")])
assert _PIV_DT.itemsize == C.sizeof(_capi.PivotRec)


def _result(handle, M, N, dtype, path=None) -> AlignmentResult:
    """The Python result of one C result handle; `path` (optional) is a
    preallocated (path_len, 2) int64 array to fill."""
    L = _capi.load()
    info = _capi.AlignInfo()
    _capi.check(L.lmdtw_result_info(handle, C.byref(info)))
    if path is None:
        path = np.empty((info.path_len, 2), np.int64)
    _capi.check(L.lmdtw_result_path(handle, _capi.ptr(path)))
    recs = np.empty(max(1, info.n_pivots), _PIV_DT)
    _capi.check(L.lmdtw_result_pivots(handle, _capi.ptr(recs)))
    # the reference's key order (divide.py:160-164)
    trace = tuple(
        {"i": r[0], "j": r[1], "i_off": r[2], "j_off": r[3], "M": r[4], "N": r[5], "sub_i": r[6], "sub_j": r[7],
         "total_at_pivot": r[9], "diagonal_k": r[8]}
        for r in recs[:info.n_pivots].tolist())
    res = AlignmentResult(
        cost=float(info.cost), path=path, cells_processed=int(info.cells_processed),
        cells_budget=2 * M * N, precision=str(dtype), algorithm="linmdtw",
        peak_diag_values=int(info.peak_diag_values), peak_table_cells=int(info.peak_table_cells),
        pivot_trace=trace)  # level_stats stays () as in the reference (divide.py:203-213)
    return res


def linmdtw(X, Y, cost: str = "euclidean", config: LinMdtwConfig | None = None,
            progress=None, **overrides) -> AlignmentResult:
    """Exact DTW alignment using linear memory (divide.py:181-213).

    ``progress(cells_processed, 2*M*N)`` is called after every recursion
    level (the device's "diagonal batch") in slices of at most 1% of the
    budget, and once more at the end with the final count.
    """
    check_cost_kind(cost)
    cfg = config or LinMdtwConfig(**overrides)
    if config is not None and overrides:
        raise InvalidInputError("pass either a config object or keyword overrides, not both")
    X, Y = as_series(X), as_series(Y)
    if X.dim != Y.dim:
        raise InvalidInputError(f"feature dimension mismatch: {X.dim} vs {Y.dim}")
    M, N = len(X), len(Y)
    dtype = precision_dtype(cfg.precision)
    ccfg = _c_config(cfg)
    xf = np.ascontiguousarray(X.frames, dtype=np.float32)
    yf = np.ascontiguousarray(Y.frames, dtype=np.float32)
    errors = []

    def _cb(done, budget, _user):
        try:
            progress(int(done), int(budget))
        except BaseException as e:  # re-raised after the call returns
            errors.append(e)

    cb = _capi.PROGRESS_FN(_cb) if progress is not None else _capi.PROGRESS_FN()
    handle = C.c_void_p()
    L = _capi.load()
    _capi.check(L.lmdtw_align(_capi.get_device(), _capi.ptr(xf), M, _capi.ptr(yf), N, X.dim,
                              C.byref(ccfg), _capi.MEM_HOST, cb, None, C.byref(handle)))
    try:
        res = _result(handle, M, N, dtype)
    finally:
        L.lmdtw_result_free(handle)
    if errors:
        raise errors[0]
    return res


def align_batch(pairs, cost: str = "euclidean", config: LinMdtwConfig | None = None,
                **overrides) -> list[AlignmentResult]:
    """Exact alignments of many independent (X, Y) pairs in one fused run:
    every recursion level of every pair shares one device launch.  Each
    result equals ``linmdtw(X, Y, config=...)`` for that pair."""
    check_cost_kind(cost)
    cfg = config or LinMdtwConfig(**overrides)
    if config is not None and overrides:
        raise InvalidInputError("pass either a config object or keyword overrides, not both")
    series = [(as_series(X), as_series(Y)) for X, Y in pairs]
    if not series:
        return []
    d = series[0][0].dim
    for X, Y in series:
        if X.dim != d or Y.dim != d:
            raise InvalidInputError("all pairs must share one feature dimension")
    dtype = precision_dtype(cfg.precision)
    ccfg = _c_config(cfg)
    xs = [np.ascontiguousarray(X.frames, dtype=np.float32) for X, _ in series]
    ys = [np.ascontiguousarray(Y.frames, dtype=np.float32) for _, Y in series]
    n = len(series)
    xp = (C.c_void_p * n)(*[a.ctypes.data for a in xs])
    yp = (C.c_void_p * n)(*[a.ctypes.data for a in ys])
    Ms = (C.c_int64 * n)(*[a.shape[0] for a in xs])
    Ns = (C.c_int64 * n)(*[a.shape[0] for a in ys])
    handles = (C.c_void_p * n)()
    L = _capi.load()
    _capi.check(L.lmdtw_align_batch(_capi.get_device(), n, xp, Ms, yp, Ns, d, C.byref(ccfg),
                                    _capi.MEM_HOST, handles))
    out = []
    try:
        # every path in one allocation (one large, hugepage-eligible buffer
        # instead of n page-faulting small ones); each result holds a view
        lens = []
        for q in range(n):
            info = _capi.AlignInfo()
            _capi.check(L.lmdtw_result_info(C.c_void_p(handles[q]), C.byref(info)))
            lens.append(int(info.path_len))
        paths = np.empty((sum(lens), 2), np.int64)
        off = 0
        for q in range(n):
            out.append(_result(C.c_void_p(handles[q]), Ms[q], Ns[q], dtype, paths[off:off + lens[q]]))
            off += lens[q]
    finally:
        for q in range(n):
            L.lmdtw_result_free(C.c_void_p(handles[q]))
    return out


def cells_ratio(result: AlignmentResult, M: int, N: int) -> float:
    """Cells evaluated divided by the full-table cell count M*N (divide.py:216)."""
    return result.cells_processed / (M * N)
