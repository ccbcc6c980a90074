"""One half pass of a single strip (rows x N) for per-warp profiling."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import _capi

lib = _capi.load()
prec, d, M, N = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 12, 128, 20000)))
rng = np.random.default_rng(0)
X = rng.random((M, d), dtype=np.float32)
Y = rng.random((N, d), dtype=np.float32)
kstop = M + N - 2
dt = np.float32 if prec == 32 else np.float64
outs = [np.empty(L.diag_length(kstop - 2 + s, M, N), dt) for s in range(3)]
pd = (C.c_void_p * 3)(*[o.ctypes.data for o in outs])
cells = C.c_int64()
for rep in range(2):
    _capi.check(lib.lmdtw_half_pass(0, _capi.ptr(X), M, _capi.ptr(Y), N, d, kstop, 0, prec, 0, pd, pd,
                                    C.byref(cells)))
print("ok", cells.value)
