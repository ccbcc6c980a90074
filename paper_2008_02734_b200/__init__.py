"""B200-native exact linear-memory DTW (arXiv 2008.02734), drop-in for the
hot path of the reference package ``lmdtw``: ``linmdtw``, ``find_pivot``,
``diag_dtw`` and ``dtw_full`` with the same arguments, results and errors.

All DP arithmetic runs in hand-written sm_100a CUDA kernels behind the C ABI
in include/lmdtw_b200.h (liblmdtw_b200.so).  There is no CPU fallback.
"""
from . import _capi
from ._capi import get_device, set_device
from .core import (
    COST_KINDS,
    DEFAULT_FPS,
    AlignmentResult,
    FeatureSeries,
    InvalidInputError,
    PathValidationError,
    as_path,
    as_series,
    check_cost_kind,
    euclidean_cost,
    frame_costs,
    path_cost,
    path_costs,
    precision_dtype,
    require_valid_path,
    validate_path,
)
from .approx import (Window, coarsen, constrained_dtw, expand_window, fastdtw, mrmsdtw, project_path,
                     window_from_path)
from .diagonal import DiagBuffers, diag_cells, diag_dtw, diag_length, diag_to_grid, peak_retained_values
from .divide import LinMdtwConfig, Pivot, align_batch, cells_ratio, find_pivot, linmdtw
from .metrics import (DiscrepancyReport, discrepancy, merge_reports, proportion_below,
                      proportion_below_frames)
from .textbook import (
    DIAG,
    LEFT,
    SELF,
    TIE_DIAG_FIRST,
    TIE_LEFT_FIRST,
    UP,
    accumulated_cost_table,
    backtrace,
    dtw_full,
    tie_codes,
)

__version__ = "0.1.0"

# Loading the library is part of importing the package: a missing build is an
# ImportError, never a silent fallback.
_capi.load()

__all__ = [
    "AlignmentResult", "COST_KINDS", "DEFAULT_FPS", "DIAG", "DiagBuffers", "FeatureSeries",
    "InvalidInputError", "LEFT", "LinMdtwConfig", "PathValidationError", "Pivot", "SELF",
    "TIE_DIAG_FIRST", "TIE_LEFT_FIRST", "UP", "accumulated_cost_table", "align_batch", "as_path",
    "as_series", "backtrace", "cells_ratio", "check_cost_kind", "diag_cells", "diag_dtw",
    "diag_length", "diag_to_grid", "dtw_full", "euclidean_cost", "find_pivot", "frame_costs",
    "get_device", "linmdtw", "path_cost", "peak_retained_values", "precision_dtype",
    "require_valid_path", "set_device", "tie_codes", "validate_path",
    "Window", "coarsen", "constrained_dtw", "expand_window", "fastdtw", "mrmsdtw", "project_path",
    "window_from_path", "DiscrepancyReport", "discrepancy", "merge_reports", "proportion_below",
    "proportion_below_frames", "path_costs",
]
