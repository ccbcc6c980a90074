"""Golden vectors for the per-path steps either side of the aligner (SURVEY.md
8(f)), generated from the REAL reference.  Run here (where /root/reference
exists), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_approx.py

Writes tests/golden/approx.npz with inputs included:
  cw*  constrained_dtw (approx.py:180-220) on windows built by the reference's
       window_from_path / expand_window / Window.full, three tie rules, fp32
       and fp64, tie-heavy and gaussian features
  win* expand_window / window_from_path / project_path / coarsen outputs
  fd*  fastdtw (approx.py:223-266), md* mrmsdtw (approx.py:317-387)
  dc*  metrics.discrepancy (metrics.py:44-63)
  pc*  core.path_cost / frame_costs (core.py:167-197)
"""
from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import lmdtw  # noqa: E402  (the reference package)
from lmdtw import approx  # noqa: E402
from lmdtw.core import frame_costs, path_cost  # noqa: E402
from lmdtw.metrics import discrepancy  # noqa: E402
from lmdtw.synth import random_series, synth_pair  # noqa: E402

TIES = [("diag", "left", "up"), ("left", "diag", "up"), ("up", "left", "diag")]
MOVE = {"left": 0, "up": 1, "diag": 2}


def series(M, d, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "ties":
        return rng.integers(0, 3, size=(M, d)).astype(np.float32)
    if kind == "walk":
        return (np.cumsum(rng.standard_normal((M, d)), 0) / np.sqrt(M)).astype(np.float32)
    return rng.standard_normal((M, d)).astype(np.float32)


def main():
    out = {}
    rng = np.random.default_rng(8_2008_02734)
    n = 0
    for case in range(60):
        M, N = (int(v) for v in rng.integers(2, 400, size=2))
        d = int(rng.choice([1, 2, 4, 12, 48]))
        kind = ("ties", "gauss", "walk")[case % 3]
        X, Y = series(M, d, 100 + case, kind), series(N, d, 900 + case, kind)
        tie = TIES[case % 3]
        prec = (32, 64)[(case // 3) % 2]
        guide = lmdtw.dtw_full(X, Y, precision=64).path
        how = case % 4
        if how == 0:
            win = approx.Window.full(M, N)
        elif how == 1:
            win = approx.window_from_path(guide, int(rng.integers(0, 4)), M, N)
        elif how == 2:
            win = approx.window_from_path(guide, int(rng.integers(4, 40)), M, N)
        else:
            Mh, Nh = max(1, M // 2), max(1, N // 2)
            if min(M, N) >= 4:
                half = lmdtw.dtw_full(approx.coarsen(X), approx.coarsen(Y), precision=64).path
                win = approx.expand_window(half, int(rng.integers(0, 6)), M, N)
            else:
                win = approx.window_from_path(guide, 1, M, N)
        r = approx.constrained_dtw(X, Y, win, tie_rule=tie, precision=prec)
        out.update({f"cw{n}/X": X, f"cw{n}/Y": Y, f"cw{n}/lo": win.lo, f"cw{n}/hi": win.hi,
                    f"cw{n}/tie": np.array([MOVE[m] for m in tie], np.int32), f"cw{n}/prec": prec,
                    f"cw{n}/cost": r.cost, f"cw{n}/path": r.path, f"cw{n}/cells": r.cells_processed})
        n += 1
    out["cw_count"] = n

    # window constructions and projections (host glue)
    n = 0
    for case in range(30):
        M, N = (int(v) for v in rng.integers(4, 600, size=2))
        X, Y = series(M, 3, 300 + case, "walk"), series(N, 3, 700 + case, "walk")
        Xc, Yc = approx.coarsen(X), approx.coarsen(Y)
        half = lmdtw.dtw_full(Xc, Yc, precision=64).path
        full = lmdtw.dtw_full(X, Y, precision=64).path
        r1, r2 = int(rng.integers(0, 8)), int(rng.integers(0, 50))
        ew = approx.expand_window(half, r1, M, N)
        wp = approx.window_from_path(full, r2, M, N)
        pp = approx.project_path(half, M, N)
        out.update({f"win{n}/X": X, f"win{n}/Y": Y, f"win{n}/Xc": Xc.frames, f"win{n}/fps": Xc.frame_rate,
                    f"win{n}/half": half, f"win{n}/full": full, f"win{n}/r1": r1, f"win{n}/r2": r2,
                    f"win{n}/ew_lo": ew.lo, f"win{n}/ew_hi": ew.hi, f"win{n}/wp_lo": wp.lo,
                    f"win{n}/wp_hi": wp.hi, f"win{n}/proj": pp,
                    f"win{n}/rad": approx._largest_radius_within(full, M, N, int(rng.integers(M + N, 8 * (M + N))))})
        n += 1
    out["win_count"] = n

    # fastdtw / mrmsdtw end to end
    n = 0
    for case in range(16):
        M, N = (int(v) for v in rng.integers(50, 3000, size=2))
        X, Y = synth_pair("random-walk", M, seed=case, warp_strength=0.3, dim=4)
        Y = random_series(N, 4, 50 + case) if case % 4 == 3 else lmdtw.as_series(
            np.resize(Y.frames, (N, 4)))
        radius = [0, 1, 5, 30][case % 4]
        prec = (64, 32)[case % 2]
        tie = TIES[case % 2]
        r = approx.fastdtw(X, Y, radius=radius, tie_rule=tie, precision=prec)
        out.update({f"fd{n}/X": X.frames, f"fd{n}/Y": Y.frames, f"fd{n}/radius": radius, f"fd{n}/prec": prec,
                    f"fd{n}/tie": np.array([MOVE[m] for m in tie], np.int32), f"fd{n}/cost": r.cost,
                    f"fd{n}/path": r.path, f"fd{n}/cells": r.cells_processed, f"fd{n}/peak": r.peak_table_cells,
                    f"fd{n}/stats": json.dumps(list(r.level_stats))})
        budget = int(rng.choice([100, 1000, 20000, M * N // 3 + 100, M * N + 5]))
        frac = float(rng.choice([0.25, 0.5, 0.75]))
        m = approx.mrmsdtw(X, Y, max_cells=budget, coarse_fraction=frac, tie_rule=tie, precision=prec)
        out.update({f"md{n}/budget": budget, f"md{n}/frac": frac, f"md{n}/cost": m.cost, f"md{n}/path": m.path,
                    f"md{n}/cells": m.cells_processed, f"md{n}/peak": m.peak_table_cells,
                    f"md{n}/stats": json.dumps(list(m.level_stats))})
        # discrepancy of the approximate paths against the exact one, both directions
        ex = lmdtw.linmdtw(X, Y, precision=64).path
        out.update({f"dc{n}/p1": r.path, f"dc{n}/p2": ex, f"dc{n}/e12": discrepancy(r.path, ex).errors,
                    f"dc{n}/e21": discrepancy(ex, m.path).errors, f"dc{n}/p3": m.path})
        # path_cost in both dtypes, frame_costs of the gathered rows
        for dt in (np.float32, np.float64):
            tag = "32" if dt == np.float32 else "64"
            out[f"pc{n}/cost{tag}"] = path_cost(X, Y, ex, dtype=dt)
            out[f"pc{n}/fc{tag}"] = frame_costs(X.frames[ex[:, 0]].astype(dt), Y.frames[ex[:, 1]].astype(dt))
        n += 1
    out["fd_count"] = n
    np.savez_compressed(os.path.join(HERE, "approx.npz"), **out)
    print("wrote", sum(1 for _ in out), "arrays")


if __name__ == "__main__":
    main()
