"""Leaf solvers on small full grids: the strip engine (dtw_full) vs the band
kernel (constrained_dtw with a full window), wall time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2008_02734_b200 as L
import bench
for (M, N, d, prec) in [(500, 500, 2, 64), (390, 390, 12, 32), (1000, 1000, 2, 64), (2000, 2000, 12, 32)]:
    X, Y = bench.latent_pair(M, N, d, seed=1)
    w = L.Window.full(M, N)
    a = L.dtw_full(X, Y, precision=prec); b = L.constrained_dtw(X, Y, w, precision=prec)
    assert a.cost == b.cost and np.array_equal(a.path, b.path)
    for name, fn in (("dtw_full", lambda: L.dtw_full(X, Y, precision=prec)),
                     ("band", lambda: L.constrained_dtw(X, Y, w, precision=prec))):
        for _ in range(3): fn()
        t = time.perf_counter(); n = 20
        for _ in range(n): fn()
        print(f"{M}x{N} d={d} fp{prec} {name:9s}: {(time.perf_counter() - t) / n * 1e3:.3f} ms", flush=True)
