"""GPU debug: locate the first wrong cell of the half-pass engine."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import paper_2008_02734_b200 as L
from oracle import oracle as O
from golden_io import cases


def first_bad(X, Y, prec, direction="forward"):
    M, N = X.shape[0], Y.shape[0]
    Xo, Yo = (X[::-1], Y[::-1]) if direction == "reverse" else (X, Y)
    D, _ = O.fill(np.ascontiguousarray(Xo), np.ascontiguousarray(Yo), precision=prec)
    for kstop in range(2, M + N - 1):
        b = L.diag_dtw(X, Y, kstop, direction, precision=prec)
        k = kstop
        i, j = L.diag_cells(k, M, N)
        got, want = b.d[2], D[i, j]
        if not np.array_equal(got, want):
            bad = np.flatnonzero(got != want)
            print(f"  kstop={kstop}: {len(bad)} bad of {len(got)}; first cells:",
                  [(int(i[q]), int(j[q]), float(got[q]), float(want[q])) for q in bad[:6]])
            return kstop
    print("  all kstops ok")
    return None


for case in cases("diag_dtw")[:12]:
    X, Y = case["X"], case["Y"]
    print("case", X.shape, Y.shape, "prec", int(case["prec"]), "rev", int(case["reverse"]), flush=True)
    first_bad(X, Y, int(case["prec"]), "reverse" if int(case["reverse"]) else "forward")

rng = np.random.default_rng(0)
for d in (1, 4, 12):
    for M, N in [(64, 64), (65, 30), (130, 40), (200, 200)]:
        X = rng.standard_normal((M, d)).astype(np.float32)
        Y = rng.standard_normal((N, d)).astype(np.float32)
        for prec in (64, 32):
            print("rand", M, N, d, prec, flush=True)
            first_bad(X, Y, prec)
