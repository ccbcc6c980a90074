"""One saturated independent-strip launch for profiling: tau3.py prec d k"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2008_02734_b200 import _capi

lib = _capi.load()
prec, d, k = (int(v) for v in sys.argv[1:4])
lib.lmdtw_debug_wave_independent.argtypes = [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                             C.POINTER(C.c_double)]
ms = C.c_double()
_capi.check(lib.lmdtw_debug_wave_independent(0, prec, d, k, 8000, 1, C.byref(ms)))
print(ms.value)
