"""Anti-diagonal half pass (drop-in for the reference's diagonal module,
/root/reference/pkg/src/lmdtw/diagonal.py).

Cells on diagonal k are ordered by increasing j: idx -> (i, j) with
i = min(k, M-1) - idx and j = k - i (diagonal.py:9-10).  The values are
produced by the strip-wavefront kernel of liblmdtw_b200.so; only the last
three diagonals ever leave the device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from .core import InvalidInputError, as_series, check_cost_kind, precision_bits, precision_dtype


def diag_length(k: int, M: int, N: int) -> int:
    """Number of grid cells on anti-diagonal k of an M x N grid (diagonal.py:29)."""
    if not (0 <= k <= M + N - 2):
        raise InvalidInputError(f"diagonal {k} out of range for {M}x{N}")
    return min(k, M - 1, N - 1, M + N - 2 - k) + 1


def diag_to_grid(k: int, idx: int, M: int, N: int) -> tuple[int, int]:
    """Grid coordinates of position idx on diagonal k (diagonal.py:36)."""
    if not (0 <= idx < diag_length(k, M, N)):
        raise InvalidInputError(f"idx {idx} out of range on diagonal {k} of {M}x{N}")
    i = min(k, M - 1) - idx
    return i, k - i


def diag_cells(k: int, M: int, N: int) -> tuple[np.ndarray, np.ndarray]:
    """Vectorized (i, j) arrays for every cell on diagonal k (diagonal.py:44)."""
    L = diag_length(k, M, N)
    i = min(k, M - 1) - np.arange(L)
    return i, k - i


def peak_retained_values(kstop: int, M: int, N: int) -> int:
    """Most accumulated+raw diagonal values live at once during a run to kstop
    (diagonal.py:160-169), in closed form."""
    return int(_capi.load().lmdtw_peak_retained_values(kstop, M, N))


@dataclass(frozen=True)
class DiagBuffers:
    """Engine state after processing diagonals 0..k_last (diagonal.py:51-71)."""

    d: tuple
    c: tuple
    k_last: int
    M: int
    N: int
    reverse: bool
    cells_processed: int
    peak_values: int

    def diagonal_index(self, buffer_slot: int) -> int:
        return self.k_last - 2 + buffer_slot


def _frames(S) -> np.ndarray:
    return np.ascontiguousarray(S.frames, dtype=np.float32)


def diag_dtw(X, Y, kstop: int, direction: str = "forward", cost: str = "euclidean",
             precision=64, parallel: bool = False, on_cells=None) -> DiagBuffers:
    """Run diagonals 0..kstop on the GPU (diagonal.py:172-223).

    ``parallel`` is accepted for signature compatibility; the device schedule
    is always parallel and bit-identical to the sequential reference.
    ``on_cells`` receives incremental cell counts summing to the total.
    """
    check_cost_kind(cost)
    X, Y = as_series(X), as_series(Y)
    if X.dim != Y.dim:
        raise InvalidInputError(f"feature dimension mismatch: {X.dim} vs {Y.dim}")
    M, N = len(X), len(Y)
    if direction not in ("forward", "reverse"):
        raise InvalidInputError(f"direction must be forward or reverse, got {direction!r}")
    if not (2 <= kstop <= M + N - 2):
        raise InvalidInputError(f"kstop={kstop} out of range [2, {M + N - 2}] for {M}x{N}")
    dtype = precision_dtype(precision)
    xf, yf = _frames(X), _frames(Y)
    outs_d = [np.empty(diag_length(kstop - 2 + s, M, N), dtype) for s in range(3)]
    outs_c = [np.empty(diag_length(kstop - 2 + s, M, N), dtype) for s in range(3)]
    pd = (C.c_void_p * 3)(*[o.ctypes.data for o in outs_d])
    pc = (C.c_void_p * 3)(*[o.ctypes.data for o in outs_c])
    cells = C.c_int64()
    _capi.check(_capi.load().lmdtw_half_pass(
        _capi.get_device(), _capi.ptr(xf), M, _capi.ptr(yf), N, X.dim, int(kstop),
        1 if direction == "reverse" else 0, precision_bits(precision), _capi.MEM_HOST,
        pd, pc, C.byref(cells)))
    if on_cells is not None:
        on_cells(1)
        if cells.value > 1:
            on_cells(cells.value - 1)
    return DiagBuffers(d=tuple(outs_d), c=tuple(outs_c), k_last=int(kstop), M=M, N=N,
                       reverse=(direction == "reverse"), cells_processed=int(cells.value),
                       peak_values=peak_retained_values(kstop, M, N))
