"""Small workloads for compute-sanitizer (racecheck / synccheck / memcheck):
    compute-sanitizer --tool racecheck python tools/probes/sanitize_case.py {align,shard}
align: linmdtw (half passes, pivots, leaves, backtrace) in fp32 and fp64;
shard: one half pass cut into 3 concurrent strip shards whose first strips
read the previous shard's handoff buffer (the multi-GPU handoff protocol)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2008_02734_b200 as L  # noqa: E402
from paper_2008_02734_b200 import _capi  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "align"
X, Y = bench.chroma_pair(700, 600, 12, seed=3)
if what == "align":
    for prec in (32, 64):
        r = L.linmdtw(X, Y, min_dim=200, precision=prec)
        print("align", prec, r.cost, len(r.pivot_trace))
    Xw, Yw = bench.latent_pair(500, 450, 100, seed=4)
    for prec in (32, 64):  # WIDE kernels (cp.async-staged X / Y blocks)
        r = L.linmdtw(Xw, Yw, min_dim=200, precision=prec)
        print("align wide", prec, r.cost)
else:
    lib = _capi.load()
    M, N, d = 700, 600, 12
    kstop = (M + N) // 2
    for prec in (32, 64):
        dt = np.float32 if prec == 32 else np.float64
        lens = [L.diag_length(kstop - 2 + s, M, N) for s in range(3)]
        od = [np.zeros(max(n, 1), dt) for n in lens]
        oc = [np.zeros(max(n, 1), dt) for n in lens]
        pd = (C.c_void_p * 3)(*[o.ctypes.data for o in od])
        pc = (C.c_void_p * 3)(*[o.ctypes.data for o in oc])
        _capi.check(lib.lmdtw_debug_sharded_half_pass(0, _capi.ptr(X), C.c_int64(M), _capi.ptr(Y), C.c_int64(N), d,
                                                      C.c_int64(kstop), 0, prec, 3, pd, pc))
        ref = L.diag_dtw(X, Y, kstop, precision=prec)
        print("shard", prec, all(np.array_equal(od[s][:lens[s]], ref.d[s]) for s in range(3)))
