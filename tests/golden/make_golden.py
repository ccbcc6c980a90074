"""Generate golden vectors from the REAL reference implementation.

Run here (where /root/reference exists), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Each fixture stores its inputs, so the GPU box
needs neither the reference nor numba to replay it.  The oracle is pinned
against these (tests/test_oracle_golden.py) and the CUDA path is checked
against both (tests/test_gpu_parity.py).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import lmdtw  # noqa: E402  (the reference package)
from lmdtw.oracle import accumulated_cost_table  # noqa: E402
from lmdtw.synth import random_series, synth_pair  # noqa: E402


def _pack(store, key, **kw):
    for k, v in kw.items():
        store[f"{key}/{k}"] = np.asarray(v)


def tie_heavy(M, d, seed):
    """Small-integer features: many exact ties in costs and accumulated costs."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 3, size=(M, d)).astype(np.float32)


def gen_diag():
    out = {}
    n = 0
    # reference known answers (test_diagonal.py:49-55)
    for X, Y, kstop in (([0, 3], [0, 1, 3], 3), ([0, 1, 2], [0, 1, 2], 2)):
        Xa = np.asarray(X, np.float32)[:, None]
        Ya = np.asarray(Y, np.float32)[:, None]
        for prec in (32, 64):
            for direction in ("forward", "reverse"):
                b = lmdtw.diag_dtw(Xa, Ya, kstop, direction, precision=prec)
                _pack(out, f"c{n}", X=Xa, Y=Ya, kstop=kstop, prec=prec, reverse=int(direction == "reverse"),
                      d0=b.d[0], d1=b.d[1], d2=b.d[2], c0=b.c[0], c1=b.c[1], c2=b.c[2],
                      cells=b.cells_processed, peak=b.peak_values)
                n += 1
    rng = np.random.default_rng(20261017)
    for case in range(40):
        M, N = (int(v) for v in rng.integers(2, 300, size=2))
        d = int(rng.choice([1, 2, 3, 4, 5, 12, 16, 48]))
        if case % 5 == 4:
            X, Y = tie_heavy(M, d, case), tie_heavy(N, d, case + 1000)
        else:
            X = random_series(M, d, case).frames
            Y = random_series(N, d, case + 500).frames
        kstop = int(rng.integers(2, M + N - 1))
        prec = (32, 64)[case % 2]
        direction = ("forward", "reverse")[(case // 2) % 2]
        b = lmdtw.diag_dtw(X, Y, kstop, direction, precision=prec)
        _pack(out, f"c{n}", X=X, Y=Y, kstop=kstop, prec=prec, reverse=int(direction == "reverse"),
              d0=b.d[0], d1=b.d[1], d2=b.d[2], c0=b.c[0], c1=b.c[1], c2=b.c[2],
              cells=b.cells_processed, peak=b.peak_values)
        n += 1
    out["count"] = np.asarray(n)
    return out


def gen_full():
    out = {}
    n = 0
    hand = [([0, 3], [0, 1, 3]), ([0], [0, 1, 3]), ([5], [5]), ([0, 1, 2], [0, 1, 2]),
            ([0, 0, 1, 1], [0, 1]), ([1, 1, 1], [1, 1, 1, 1])]
    cases = [(np.asarray(a, np.float32)[:, None], np.asarray(b, np.float32)[:, None]) for a, b in hand]
    rng = np.random.default_rng(777)
    for case in range(24):
        M, N = (int(v) for v in rng.integers(1, 120, size=2))
        d = int(rng.choice([1, 2, 3, 4, 12]))
        if case % 3 == 2:
            cases.append((tie_heavy(M, d, case), tie_heavy(N, d, case + 50)))
        else:
            cases.append((random_series(M, d, case).frames, random_series(N, d, case + 99).frames))
    for X, Y in cases:
        for prec in (32, 64):
            for tname, tie in (("diag_first", lmdtw.TIE_DIAG_FIRST), ("left_first", lmdtw.TIE_LEFT_FIRST),
                               ("up_first", ("up", "left", "diag"))):
                r = lmdtw.dtw_full(X, Y, tie_rule=tie, precision=prec)
                _pack(out, f"c{n}", X=X, Y=Y, prec=prec, tie=np.array([{"left": 0, "up": 1, "diag": 2}[m] for m in tie]),
                      cost=r.cost, path=r.path)
                if X.shape[0] * Y.shape[0] <= 4000 and tname == "diag_first":
                    out[f"c{n}/table"] = accumulated_cost_table(X, Y, precision=prec)
                n += 1
    out["count"] = np.asarray(n)
    return out


def gen_pivot():
    out = {}
    n = 0
    hand = [([0, 3], [0, 1, 3]), ([0, 1, 2, 4, 7, 11], [0, 1, 2, 4, 7, 11]), ([1, 1, 1, 1], [1, 1, 1])]
    cases = [(np.asarray(a, np.float32)[:, None], np.asarray(b, np.float32)[:, None]) for a, b in hand]
    rng = np.random.default_rng(4242)
    for case in range(30):
        M, N = (int(v) for v in rng.integers(2, 250, size=2))
        if M + N - 2 < 2:
            continue
        d = int(rng.choice([1, 2, 3, 8, 12]))
        if case % 3 == 0:
            cases.append((tie_heavy(M, d, case), tie_heavy(N, d, case + 7)))
        else:
            cases.append((random_series(M, d, case).frames, random_series(N, d, case + 31).frames))
    for X, Y in cases:
        for prec in (32, 64):
            for rule in ("lowest", "highest"):
                p = lmdtw.find_pivot(X, Y, precision=prec, pivot_tie_rule=rule)
                _pack(out, f"c{n}", X=X, Y=Y, prec=prec, highest=int(rule == "highest"),
                      i=p.i, j=p.j, total=p.total_at_pivot, k=p.diagonal_k)
                n += 1
    out["count"] = np.asarray(n)
    return out


def _trace_arrays(trace):
    keys = ("i", "j", "i_off", "j_off", "M", "N", "sub_i", "sub_j", "diagonal_k")
    ints = np.array([[e[k] for k in keys] for e in trace], dtype=np.int64).reshape(-1, len(keys))
    tots = np.array([e["total_at_pivot"] for e in trace], dtype=np.float64)
    return ints, tots


def gen_linmdtw():
    out = {}
    n = 0
    cases = []
    A, B = synth_pair("random-walk", 1000, seed=0, warp_strength=0.3, dim=2)  # BASELINE cfg1
    for prec in (64, 32):
        cases.append((A.frames, B.frames, dict(precision=prec)))
    cases.append((np.asarray([[0], [3]], np.float32), np.asarray([[0], [1], [3]], np.float32), dict(min_dim=2)))
    cases.append((np.asarray([[0]], np.float32), np.asarray([[0], [1], [3]], np.float32), dict(min_dim=2)))
    X, Y = random_series(400, 8, 11).frames, random_series(350, 8, 12).frames
    cases.append((X, Y, dict(min_dim=16)))
    cases.append((X, Y, dict(min_dim=16, precision=32)))
    X, Y = synth_pair("warped-sine", 220, seed=5, warp_strength=0.3)
    cases.append((X.frames, Y.frames, dict(min_dim=16)))
    rng = np.random.default_rng(99)
    for case in range(14):
        M, N = (int(v) for v in rng.integers(2, 400, size=2))
        d = int(rng.choice([1, 2, 4, 12]))
        md = int(rng.choice([2, 4, 16, 64]))
        prec = (64, 32)[case % 2]
        rule = ("lowest", "highest")[(case // 2) % 2]
        tie = (lmdtw.TIE_DIAG_FIRST, lmdtw.TIE_LEFT_FIRST)[(case // 4) % 2]
        if case % 3 == 0:
            X, Y = tie_heavy(M, d, case), tie_heavy(N, d, case + 3)
        else:
            X, Y = random_series(M, d, case + 5).frames, random_series(N, d, case + 6).frames
        cases.append((X, Y, dict(min_dim=md, precision=prec, pivot_tie_rule=rule, tie_rule=tie)))
    for X, Y, kw in cases:
        r = lmdtw.linmdtw(X, Y, **kw)
        ints, tots = _trace_arrays(r.pivot_trace)
        tie = kw.get("tie_rule", lmdtw.TIE_DIAG_FIRST)
        _pack(out, f"c{n}", X=X, Y=Y, prec=kw.get("precision", 64), min_dim=kw.get("min_dim", 500),
              highest=int(kw.get("pivot_tie_rule", "lowest") == "highest"),
              tie=np.array([{"left": 0, "up": 1, "diag": 2}[m] for m in tie]),
              cost=r.cost, path=r.path, cells=r.cells_processed, peak_diag=r.peak_diag_values,
              peak_table=r.peak_table_cells, piv_ints=ints, piv_tot=tots)
        n += 1
    out["count"] = np.asarray(n)
    return out


def main():
    for name, fn in (("diag_dtw", gen_diag), ("dtw_full", gen_full), ("find_pivot", gen_pivot),
                     ("linmdtw", gen_linmdtw)):
        data = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path}: {int(data['count'])} cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    sys.exit(main())
