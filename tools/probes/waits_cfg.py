"""Blocked mbarrier-wait cycles by tag for one alignment of a bench config
(LMDTW_WAITSTATS build):  python tools/probes/waits_cfg.py cfg1"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import _capi
lib = _capi.load()
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
X, Y = bench.make_inputs(name)[0]
prec = bench.CONFIGS[name]["prec"]
for _ in range(3):
    L.linmdtw(X, Y, precision=prec)
cyc = (C.c_ulonglong * 16)(); cnt = (C.c_ulonglong * 16)()
lib.lmdtw_debug_wait_stats(cyc, cnt, 1)
L.linmdtw(X, Y, precision=prec)
lib.lmdtw_debug_wait_stats(cyc, cnt, 0)
names = {1: "item queue (cost)", 2: "Y TMA (cost)", 3: "ring empty (cost)", 4: "pad (cost)", 5: "item (DP)",
         6: "ring full (DP)", 7: "pad (DP)"}
for t in range(16):
    if cnt[t]:
        print(f"tag {t} {names.get(t, '?'):20s}: {cnt[t]:9d} waits, {cyc[t] / 1.965e3:10.1f} us summed over warps")
