"""Per-warp step time of the strip engine: full-grid half passes of
k strips x N columns; reports kernel time / steps."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import _capi

lib = _capi.load()
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 32
d = int(sys.argv[2]) if len(sys.argv) > 2 else 12
H = 128 if prec == 32 else 64
N = 20000
rng = np.random.default_rng(0)
Y = rng.random((N, d), dtype=np.float32)
_capi.profile(True)
for k in (1, 2, 8, 148, 296, 592, 1184, 2368):
    M = H * k
    X = rng.random((M, d), dtype=np.float32)
    kstop = M + N - 2
    dt = np.float32 if prec == 32 else np.float64
    outs = [np.empty(L.diag_length(kstop - 2 + s, M, N), dt) for s in range(3)]
    pd = (C.c_void_p * 3)(*[o.ctypes.data for o in outs])
    pc = (C.c_void_p * 3)(*[o.ctypes.data for o in outs])
    cells = C.c_int64()
    for rep in range(2):
        _capi.profile_reset()
        _capi.check(lib.lmdtw_half_pass(0, _capi.ptr(X), M, _capi.ptr(Y), N, d, kstop, 0, prec, 0, pd, pc,
                                        C.byref(cells)))
    p = _capi.profile_get()
    ms = p["wave_ms"]
    print(f"strips={k:5d} rows={M:7d} N={N} kernel {ms:8.3f} ms  tau={ms * 1e-3 * 1.965e9 / N:7.1f} cyc/step "
          f"(at 1.965GHz)  {cells.value / ms / 1e6:8.1f} Gcell/s", flush=True)
