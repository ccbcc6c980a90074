"""One launch set of independent single-strip passes (for ncu): args prec d npasses N."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2008_02734_b200 import _capi

lib = _capi.load()
prec, d, n, N = (int(v) for v in sys.argv[1:5])
ms = C.c_double()
_capi.check(lib.lmdtw_debug_wave_independent(0, prec, d, n, N, 1, C.byref(ms)))
print(f"{n} strips x {N}: {ms.value:.3f} ms, {ms.value * 1e-3 * 1.965e9 / (N + 31):.1f} cyc/step")
