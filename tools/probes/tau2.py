"""Strip-engine step rate with independent strips (no handoff chains)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2008_02734_b200 import _capi

lib = _capi.load()
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 32
d = int(sys.argv[2]) if len(sys.argv) > 2 else 12
R = (4 if d <= 32 else 2) if prec == 32 else (2 if d <= 16 else 1)
N = 8000
lib.lmdtw_debug_wave_independent.argtypes = [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                             C.POINTER(C.c_double)]
for k in (1, 148, 296, 592, 1184, 1776, 2368, 4736):
    ms = C.c_double()
    _capi.check(lib.lmdtw_debug_wave_independent(0, prec, d, k, N, 3, C.byref(ms)))
    cells = k * 32 * R * N
    print(f"prec={prec} d={d} strips={k:5d} {ms.value:8.3f} ms  step={ms.value * 1e-3 * 1.965e9 / N:7.1f} cyc "
          f"(1.965GHz)  {cells / ms.value / 1e6:8.1f} Gcell/s", flush=True)
