import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import paper_2008_02734_b200 as L
from oracle import oracle as O
from golden_io import cases
for case in cases("diag_dtw")[:8]:
    X, Y = case["X"], case["Y"]
    dr = "reverse" if int(case["reverse"]) else "forward"
    b = L.diag_dtw(X, Y, int(case["kstop"]), dr, precision=int(case["prec"]))
    print(X.ravel()[:4], Y.ravel()[:4], int(case["kstop"]), dr, int(case["prec"]))
    for s in range(3):
        print("  slot", s, "got", b.d[s], b.c[s], "want", case[f"d{s}"], case[f"c{s}"])
