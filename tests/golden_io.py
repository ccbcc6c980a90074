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


def acceptance_c1():
    """Criterion-1 sweep records (tests/golden/make_acceptance.py): per instance
    the inputs (regenerated from the seeds as the reference's random_series
    does), the certified minimum cost, and the reference's linmdtw result
    (cost, path, pivot trace) in fp32 and fp64."""
    with np.load(os.path.join(GOLDEN, "acceptance_c1.npz")) as f:
        z = {k: f[k] for k in f.files}  # npz members decompress on every access
    keys = ("i", "j", "i_off", "j_off", "M", "N", "sub_i", "sub_j", "diagonal_k")
    out = []
    po = {32: 0, 64: 0}
    vo = {32: 0, 64: 0}
    for q, (dim, M, N, rep, seed) in enumerate(z["meta"]):
        X = np.random.default_rng(int(seed)).standard_normal((int(M), int(dim))).astype(np.float32)
        Y = np.random.default_rng(int(seed) + 7).standard_normal((int(N), int(dim))).astype(np.float32)
        rec = {"X": X, "Y": Y, "dag_cost": float(z["dag_cost"][q])}
        for prec in (32, 64):
            n = int(z[f"plen{prec}"][q])
            path = z[f"path{prec}"][po[prec]:po[prec] + n].astype(np.int64)
            po[prec] += n
            k = int(z[f"npiv{prec}"][q])
            trace = []
            for row, tot in zip(z[f"piv{prec}"][vo[prec]:vo[prec] + k], z[f"ptot{prec}"][vo[prec]:vo[prec] + k]):
                e = {kk: int(v) for kk, v in zip(keys, row)}
                e["total_at_pivot"] = float(tot)
                trace.append(e)
            vo[prec] += k
            rec[prec] = {"cost": float(z[f"cost{prec}"][q]), "path": path, "trace": trace}
        out.append(rec)
    return out


_APPROX = None


def approx_cases(prefix):
    """Records of tests/golden/approx.npz (make_golden_approx.py) whose keys
    start with `prefix` ("cw", "win", "fd", "md", "dc", "pc"); md/dc/pc records
    share the index of the fd record built from the same inputs."""
    global _APPROX
    if _APPROX is None:
        with np.load(os.path.join(GOLDEN, "approx.npz")) as f:
            _APPROX = {k: f[k] for k in f.files}
    count = int(_APPROX[("fd" if prefix in ("md", "dc", "pc") else prefix) + "_count"])
    out = []
    for q in range(count):
        pre = f"{prefix}{q}/"
        out.append({k[len(pre):]: v for k, v in _APPROX.items() if k.startswith(pre)})
    return out
