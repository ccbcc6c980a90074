"""Pace of independent single-strip passes (no strip-to-strip coupling):
npasses strips of H rows x N columns run concurrently; cycles per DP step."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2008_02734_b200 import _capi

lib = _capi.load()
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 32
d = int(sys.argv[2]) if len(sys.argv) > 2 else 12
N = 20000
for n in (1, 2, 4, 8, 148, 296, 444, 592, 1184):
    ms = C.c_double()
    _capi.check(lib.lmdtw_debug_wave_independent(0, prec, d, n, N, 5, C.byref(ms)))
    cyc = ms.value * 1e-3 * 1.965e9 / (N + 31)
    H = int(lib.lmdtw_strip_height(prec, d))
    cells = n * H * N
    print(f"independent strips={n:5d}: {ms.value:8.3f} ms  {cyc:7.1f} cyc/step  {cells / ms.value / 1e6:8.1f} Gcell/s",
          flush=True)
