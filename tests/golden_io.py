"""Load the golden fixtures written by tests/golden/make_golden.py."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MOVES = {0: "left", 1: "up", 2: "diag"}


def cases(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    n = int(z["count"])
    out = []
    for q in range(n):
        pre = f"c{q}/"
        out.append({k[len(pre):]: z[k] for k in z.files if k.startswith(pre)})
    return out


def tie_rule(codes):
    return tuple(MOVES[int(c)] for c in codes)


def trace_from(case):
    keys = ("i", "j", "i_off", "j_off", "M", "N", "sub_i", "sub_j", "diagonal_k")
    ints = case["piv_ints"].reshape(-1, len(keys))
    out = []
    for row, tot in zip(ints, case["piv_tot"]):
        e = {k: int(v) for k, v in zip(keys, row)}
        e["total_at_pivot"] = float(tot)
        out.append(e)
    return out
