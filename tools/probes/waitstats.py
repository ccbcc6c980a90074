"""Blocked-wait cycles per mbarrier tag for an independent-strip run (LMDTW_WAITSTATS build)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2008_02734_b200 import _capi
lib = _capi.load()
cyc = (C.c_ulonglong * 16)(); cnt = (C.c_ulonglong * 16)()
ms = C.c_double()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
_capi.check(lib.lmdtw_debug_wave_independent(0, 32, 12, n, 20000, 1, C.byref(ms)))
lib.lmdtw_debug_wait_stats(cyc, cnt, 1)
_capi.check(lib.lmdtw_debug_wave_independent(0, 32, 12, n, 20000, 1, C.byref(ms)))
lib.lmdtw_debug_wait_stats(cyc, cnt, 0)
# the second call ran 3 launches after the reset (2 warm-up + 1 timed)
names = {1: "item queue (cost)", 2: "Y TMA (cost)", 3: "ring empty (cost)", 5: "item (DP)", 6: "ring full (DP)", 7: "pad (DP)", 4: "pad (cost)"}
kcyc = ms.value * 1e-3 * 1.965e9
print(f"{n} strips: {ms.value:.3f} ms per launch ({kcyc:.3g} cycles)")
for t in range(16):
    if cnt[t]:
        per_warp = cyc[t] / 3 / (n * (3 if t in (1, 2, 3, 4) else 1))
        print(f"  tag {t} {names.get(t, '?'):20s}: waits {cnt[t] // 3:9d}, {per_warp / kcyc * 100:5.1f}% of each such warp's time")
