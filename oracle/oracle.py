"""ctypes front end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  The product package (paper_2008_02734_b200)
never does.  The C restatement lives in lmdtw_oracle.c and cites the reference
file:line for every function; its parity pin is tests/test_oracle_golden.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblmdtw_oracle.so")
_lib = None

LEFT, UP, DIAG, SELF = 0, 1, 2, 3
_MOVE = {"left": LEFT, "up": UP, "diag": DIAG}


class OrcPivot(C.Structure):
    _fields_ = [("i", C.c_int64), ("j", C.c_int64), ("i_off", C.c_int64), ("j_off", C.c_int64),
                ("M", C.c_int64), ("N", C.c_int64), ("sub_i", C.c_int64), ("sub_j", C.c_int64),
                ("diagonal_k", C.c_int64), ("total_at_pivot", C.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (OpenMP if available, else serial)."""
    src = os.path.join(_HERE, "lmdtw_oracle.c")
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src):
        return _LIB_PATH
    base = ["gcc", "-O2", "-fPIC", "-ffp-contract=off", "-fno-math-errno", "-std=c11", "-shared",
            "-o", _LIB_PATH, src, "-lm"]
    try:
        subprocess.run(base[:1] + ["-fopenmp"] + base[1:], check=True, capture_output=True)
    except subprocess.CalledProcessError:
        subprocess.run(base, check=True, capture_output=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P, I64, I = C.c_void_p, C.c_int64, C.c_int
        L.orc_diag_length.argtypes = [I64, I64, I64]
        L.orc_diag_length.restype = I64
        L.orc_peak_retained_values.argtypes = [I64, I64, I64]
        L.orc_peak_retained_values.restype = I64
        for sfx in ("f32", "f64"):
            f = getattr(L, f"orc_half_pass_{sfx}")
            f.argtypes = [P, I64, P, I64, I64, I64, I, I64, P, P]
            f.restype = I64
            f = getattr(L, f"orc_dtw_fill_{sfx}")
            f.argtypes = [P, I64, P, I64, I64, I64, I, P, P, P]
            f.restype = None
            f = getattr(L, f"orc_dtw_full_{sfx}")
            f.argtypes = [P, I64, P, I64, I64, I64, I, P, P, P]
            f.restype = I64
            f = getattr(L, f"orc_find_pivot_{sfx}")
            f.argtypes = [P, P, I64, I64, I, I, P, P, P, P, P, P]
            f.restype = I
            f = getattr(L, f"orc_window_dtw_{sfx}")
            f.argtypes = [P, P, I64, I64, I, P, P, P, P, P, P]
            f.restype = I64
            f = getattr(L, f"orc_path_cost_{sfx}")
            f.argtypes = [P, P, I, P, I64]
            f.restype = C.c_double
        L.orc_linmdtw.argtypes = [P, P, I64, I64, I, I, I, P, I, I, P, P, P, P, P, P, P]
        L.orc_linmdtw.restype = I64
        L.orc_free.argtypes = [P]
        L.orc_num_threads.restype = I
        _lib = L
    return _lib


def _f32(a):
    a = np.asarray(a, dtype=np.float32)
    if a.ndim == 1:
        a = a[:, None]
    return np.ascontiguousarray(a)


def _sfx(precision):
    return "f32" if int(precision) == 32 else "f64"


def _dt(precision):
    return np.float32 if int(precision) == 32 else np.float64


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def tie_codes(tie_rule):
    return np.array([_MOVE[m] for m in tie_rule], dtype=np.int32)


def diag_length(k, M, N):
    return int(lib().orc_diag_length(k, M, N))


def peak_retained_values(kstop, M, N):
    return int(lib().orc_peak_retained_values(kstop, M, N))


def half_pass(X, Y, kstop, direction="forward", precision=64):
    """Oracle diag_dtw: returns (d tuple, c tuple, cells_processed)."""
    X, Y = _f32(X), _f32(Y)
    M, N, d = X.shape[0], Y.shape[0], X.shape[1]
    dt = _dt(precision)
    outs_d = [np.empty(diag_length(kstop - 2 + s, M, N), dt) for s in range(3)]
    outs_c = [np.empty(diag_length(kstop - 2 + s, M, N), dt) for s in range(3)]
    pd = (C.c_void_p * 3)(*[o.ctypes.data for o in outs_d])
    pc = (C.c_void_p * 3)(*[o.ctypes.data for o in outs_c])
    if direction == "reverse":
        xb = X.ctypes.data + (M - 1) * d * 4
        yb = Y.ctypes.data + (N - 1) * d * 4
        cells = getattr(lib(), f"orc_half_pass_{_sfx(precision)}")(xb, -d, yb, -d, M, N, d, kstop, pd, pc)
    else:
        cells = getattr(lib(), f"orc_half_pass_{_sfx(precision)}")(_ptr(X), d, _ptr(Y), d, M, N, d, kstop, pd, pc)
    return tuple(outs_d), tuple(outs_c), int(cells)


def fill(X, Y, tie_rule=("diag", "left", "up"), precision=64):
    """Oracle _dtw_fill: full (D, P) tables."""
    X, Y = _f32(X), _f32(Y)
    M, N, d = X.shape[0], Y.shape[0], X.shape[1]
    D = np.empty((M, N), _dt(precision))
    P = np.empty((M, N), np.uint8)
    tie = tie_codes(tie_rule)
    getattr(lib(), f"orc_dtw_fill_{_sfx(precision)}")(_ptr(X), d, _ptr(Y), d, M, N, d, _ptr(tie), _ptr(D), _ptr(P))
    return D, P


def dtw_full(X, Y, tie_rule=("diag", "left", "up"), precision=64):
    """Oracle dtw_full: (cost, path)."""
    X, Y = _f32(X), _f32(Y)
    M, N, d = X.shape[0], Y.shape[0], X.shape[1]
    path = np.empty((M + N - 1, 2), np.int64)
    cost = C.c_double()
    tie = tie_codes(tie_rule)
    n = getattr(lib(), f"orc_dtw_full_{_sfx(precision)}")(_ptr(X), d, _ptr(Y), d, M, N, d, _ptr(tie),
                                                          C.byref(cost), _ptr(path))
    if n < 0:
        raise RuntimeError(f"oracle dtw_full failed ({n})")
    return cost.value, path[:n].copy()


def find_pivot(X, Y, precision=64, pivot_tie_rule="lowest"):
    """Oracle find_pivot: dict(i, j, total_at_pivot, diagonal_k, cells, peak)."""
    X, Y = _f32(X), _f32(Y)
    M, N, d = X.shape[0], Y.shape[0], X.shape[1]
    pi, pj, k, cells, peak = (C.c_int64() for _ in range(5))
    tot = C.c_double()
    rc = getattr(lib(), f"orc_find_pivot_{_sfx(precision)}")(
        _ptr(X), _ptr(Y), M, N, d, 1 if pivot_tie_rule == "highest" else 0,
        C.byref(pi), C.byref(pj), C.byref(tot), C.byref(k), C.byref(cells), C.byref(peak))
    if rc != 0:
        raise ValueError("too small for a pivot search")
    return dict(i=pi.value, j=pj.value, total_at_pivot=tot.value, diagonal_k=k.value,
                cells=cells.value, peak=peak.value)


def window_dtw(X, Y, lo, hi, tie_rule=("diag", "left", "up"), precision=64):
    """Oracle constrained_dtw over the window lo/hi: (cost, path, cells)."""
    X, Y = _f32(X), _f32(Y)
    M, N, d = X.shape[0], Y.shape[0], X.shape[1]
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    path = np.empty((M + N - 1, 2), np.int64)
    cost = C.c_double()
    cells = C.c_int64()
    tie = tie_codes(tie_rule)
    n = getattr(lib(), f"orc_window_dtw_{_sfx(precision)}")(_ptr(X), _ptr(Y), M, N, d, _ptr(lo), _ptr(hi),
                                                            _ptr(tie), C.byref(cost), _ptr(path), C.byref(cells))
    if n < 0:
        raise RuntimeError(f"oracle window_dtw failed ({n})")
    return cost.value, path[:n].copy(), cells.value


def path_cost(X, Y, path, precision=64):
    X, Y = _f32(X), _f32(Y)
    p = np.ascontiguousarray(np.asarray(path, dtype=np.int64))
    return float(getattr(lib(), f"orc_path_cost_{_sfx(precision)}")(_ptr(X), _ptr(Y), X.shape[1], _ptr(p), p.shape[0]))


def linmdtw(X, Y, min_dim=500, precision=64, tie_rule=("diag", "left", "up"),
            pivot_tie_rule="lowest", nthreads=1):
    """Oracle linmdtw: dict(cost, path, cells_processed, peak_diag_values,
    peak_table_cells, pivot_trace)."""
    X, Y = _f32(X), _f32(Y)
    M, N, d = X.shape[0], Y.shape[0], X.shape[1]
    path = np.empty((M + N - 1, 2), np.int64)
    cost = C.c_double()
    cells, pk_d, pk_t, npiv = (C.c_int64() for _ in range(4))
    piv = C.POINTER(OrcPivot)()
    tie = tie_codes(tie_rule)
    n = lib().orc_linmdtw(_ptr(X), _ptr(Y), M, N, d, int(precision), int(min_dim), _ptr(tie),
                          1 if pivot_tie_rule == "highest" else 0, int(nthreads), _ptr(path),
                          C.byref(cost), C.byref(cells), C.byref(pk_d), C.byref(pk_t),
                          C.byref(piv), C.byref(npiv))
    if n < 0:
        raise RuntimeError(f"oracle linmdtw failed ({n})")
    trace = []
    for q in range(npiv.value):
        p = piv[q]
        trace.append({"i": p.i, "j": p.j, "i_off": p.i_off, "j_off": p.j_off, "M": p.M, "N": p.N,
                      "sub_i": p.sub_i, "sub_j": p.sub_j, "total_at_pivot": p.total_at_pivot,
                      "diagonal_k": p.diagonal_k})
    if npiv.value:
        lib().orc_free(C.cast(piv, C.c_void_p))
    return dict(cost=cost.value, path=path[:n].copy(), cells_processed=cells.value,
                peak_diag_values=pk_d.value, peak_table_cells=pk_t.value, pivot_trace=tuple(trace))


def num_threads():
    return int(lib().orc_num_threads())
