"""C-ABI library checks that need no GPU: it loads, exports every symbol the
header declares, its host-side closed forms and path_cost agree with the
oracle, and compute calls fail loudly (no CPU fallback) without a device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import _capi
from golden_io import cases
from oracle import oracle as O

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "lmdtw_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(lmdtw_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(_capi.EXPORTS) <= set(syms)


def test_version_and_limits():
    lib = _capi.load()
    assert b"sm_100a" in lib.lmdtw_version()
    assert lib.lmdtw_max_dim(32) >= 48 and lib.lmdtw_max_dim(64) >= 48


def test_closed_forms_match_oracle():
    lib = _capi.load()
    rng = np.random.default_rng(0)
    for _ in range(300):
        M, N = (int(v) for v in rng.integers(1, 60, size=2))
        for k in range(-1, M + N):
            assert lib.lmdtw_diag_length(k, M, N) == O.diag_length(k, M, N)
        kstop = int(rng.integers(0, M + N - 1))
        want = sum(O.diag_length(k, M, N) for k in range(kstop + 1))
        assert lib.lmdtw_cells_upto(kstop, M, N) == want
        assert L.peak_retained_values(kstop, M, N) == O.peak_retained_values(kstop, M, N)


def test_peak_closed_form_large_shapes():
    for M, N in [(100000, 100000), (200000, 20000), (501, 500), (1000, 3), (7, 9000)]:
        K = M + N - 1
        kf = (K + 1) // 2
        assert L.peak_retained_values(kf, M, N) == O.peak_retained_values(kf, M, N)


def host_path_cost(X, Y, path, prec=64):
    """The library's host routine lmdtw_path_cost (L.path_cost runs on the GPU)."""
    import ctypes as C
    from paper_2008_02734_b200 import _capi
    X = np.ascontiguousarray(np.asarray(X, np.float32).reshape(len(X), -1))
    Y = np.ascontiguousarray(np.asarray(Y, np.float32).reshape(len(Y), -1))
    p = np.ascontiguousarray(np.asarray(path, np.int64))
    out = C.c_double()
    _capi.check(_capi.load().lmdtw_path_cost(_capi.ptr(X), len(X), _capi.ptr(Y), len(Y), X.shape[1],
                                             _capi.ptr(p), len(p), prec, C.byref(out)))
    return out.value


def test_path_cost_host_routine_matches_reference_golden():
    for case in cases("linmdtw"):
        got = host_path_cost(case["X"], case["Y"], case["path"], int(case["prec"]))
        assert got == float(case["cost"])


def test_path_cost_known_answers():
    s = lambda v: np.asarray(v, np.float32)[:, None]
    assert host_path_cost(s([0, 1, 2]), s([0, 1, 2]), [(0, 0), (1, 1), (2, 2)]) == 0.0
    assert host_path_cost(s([0, 3]), s([0, 1, 3]), [(0, 0), (0, 1), (1, 2)]) == 1.0
    assert host_path_cost(s([0]), s([0, 1, 3]), [(0, 0), (0, 1), (0, 2)]) == 4.0
    with pytest.raises(L.PathValidationError):
        L.path_cost(s([0, 3]), s([0, 1, 3]), [(0, 0), (1, 2)])


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="checks the no-device failure mode")
def test_compute_without_device_fails_loudly():
    X = np.arange(8, dtype=np.float32)[:, None]
    with pytest.raises(RuntimeError, match="no CUDA device"):
        L.linmdtw(X, X, min_dim=2)
    with pytest.raises(RuntimeError):
        L.dtw_full(X, X)
    with pytest.raises(RuntimeError):
        L.diag_dtw(X, X, kstop=4)


def test_no_contracted_packed_fma_in_sass():
    """Bit parity needs unfused mul/add.  ptxas contracts mul.rn.f32x2 +
    add.rn.f32x2 into FFMA2, so squares are written as fma(d, d, +0): every
    FFMA2 in the library must have the zero register as its addend."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True, text=True).stdout
    ffma2 = [l for l in sass.splitlines() if "FFMA2" in l]
    assert ffma2, "expected packed f32x2 squares in the fp32 kernels"
    assert all("RZ.F32" in l for l in ffma2), [l for l in ffma2 if "RZ.F32" not in l][:3]
