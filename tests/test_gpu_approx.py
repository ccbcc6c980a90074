"""GPU parity of the per-path steps either side of the aligner:
constrained_dtw's windowed DP (band_kernel), fastdtw / mrmsdtw end to end,
device path_cost / frame_costs and discrepancy -- bit-exact against the
reference's golden vectors (tests/golden/approx.npz) and the C oracle."""
import json

import numpy as np
import pytest

import bench
import paper_2008_02734_b200 as L
from golden_io import approx_cases, tie_rule
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_constrained_dtw_golden():
    for c in approx_cases("cw"):
        X, Y = c["X"], c["Y"]
        w = L.Window(c["lo"], c["hi"], Y.shape[0])
        r = L.constrained_dtw(X, Y, w, tie_rule=tie_rule(c["tie"]), precision=int(c["prec"]))
        assert r.cost == float(c["cost"])
        assert np.array_equal(r.path, c["path"])
        assert r.cells_processed == int(c["cells"]) == r.peak_table_cells
        assert r.algorithm == "constrained" and r.cells_budget == X.shape[0] * Y.shape[0]


@pytest.mark.parametrize("prec", [32, 64])
def test_constrained_dtw_large_vs_oracle(prec):
    """Long bands (the shapes fastdtw / mrmsdtw refine at): 20k x 18k chroma
    pair, windows of radius 0, 8 and 300 around the exact path, plus a full
    window on a smaller pair; tie-heavy features under the left-first rule."""
    X, Y = bench.chroma_pair(20000, 18000, 12, seed=21)
    guide = L.linmdtw(X, Y, precision=64).path
    for r in (0, 8, 300):
        w = L.window_from_path(guide, r, 20000, 18000)
        g = L.constrained_dtw(X, Y, w, precision=prec)
        cost, path, cells = O.window_dtw(X, Y, w.lo, w.hi, precision=prec)
        assert g.cost == cost and np.array_equal(g.path, path) and g.cells_processed == cells
    rng = np.random.default_rng(3)
    Xt = rng.integers(0, 3, size=(1500, 5)).astype(np.float32)
    Yt = rng.integers(0, 3, size=(1300, 5)).astype(np.float32)
    for w in (L.Window.full(1500, 1300), L.window_from_path(L.dtw_full(Xt, Yt).path, 40, 1500, 1300)):
        g = L.constrained_dtw(Xt, Yt, w, tie_rule=L.TIE_LEFT_FIRST, precision=prec)
        cost, path, cells = O.window_dtw(Xt, Yt, w.lo, w.hi, L.TIE_LEFT_FIRST, precision=prec)
        assert g.cost == cost and np.array_equal(g.path, path) and g.cells_processed == cells
    # the full window is the textbook DP
    f = L.dtw_full(Xt, Yt, tie_rule=L.TIE_LEFT_FIRST, precision=prec)
    g = L.constrained_dtw(Xt, Yt, L.Window.full(1500, 1300), tie_rule=L.TIE_LEFT_FIRST, precision=prec)
    assert g.cost == f.cost and np.array_equal(g.path, f.path)


def test_constrained_dtw_errors():
    X = np.zeros((4, 2), np.float32)
    Y = np.zeros((5, 2), np.float32)
    with pytest.raises(L.InvalidInputError, match="shape does not match"):
        L.constrained_dtw(X, Y, L.Window.full(4, 4))
    with pytest.raises(L.InvalidInputError, match="disconnected"):
        L.constrained_dtw(X, Y, L.Window(np.array([0, 3, 3, 3]), np.array([1, 4, 4, 4]), 5))


def _stats(r):
    return [dict(s) for s in r.level_stats]


def test_fastdtw_golden():
    for c in approx_cases("fd"):
        r = L.fastdtw(c["X"], c["Y"], radius=int(c["radius"]), tie_rule=tie_rule(c["tie"]),
                      precision=int(c["prec"]))
        assert r.cost == float(c["cost"])
        assert np.array_equal(r.path, c["path"])
        assert r.cells_processed == int(c["cells"]) and r.peak_table_cells == int(c["peak"])
        assert _stats(r) == json.loads(str(c["stats"]))


def test_mrmsdtw_golden():
    for f, c in zip(approx_cases("fd"), approx_cases("md")):
        r = L.mrmsdtw(f["X"], f["Y"], max_cells=int(c["budget"]), coarse_fraction=float(c["frac"]),
                      tie_rule=tie_rule(f["tie"]), precision=int(f["prec"]))
        assert r.cost == float(c["cost"])
        assert np.array_equal(r.path, c["path"])
        assert r.cells_processed == int(c["cells"]) and r.peak_table_cells == int(c["peak"])
        assert _stats(r) == json.loads(str(c["stats"]))


def test_discrepancy_golden():
    for c in approx_cases("dc"):
        assert np.array_equal(L.discrepancy(c["p1"], c["p2"]).errors, c["e12"])
        assert np.array_equal(L.discrepancy(c["p2"], c["p3"]).errors, c["e21"])


def test_path_cost_and_frame_costs_golden():
    for f, d, c in zip(approx_cases("fd"), approx_cases("dc"), approx_cases("pc")):
        X, Y, path = L.FeatureSeries(f["X"]), L.FeatureSeries(f["Y"]), d["p2"]
        assert L.path_cost(X, Y, path, dtype=np.float32) == float(c["cost32"])
        assert L.path_cost(X, Y, path, dtype=np.float64) == float(c["cost64"])
        for dt, tag in ((np.float32, "32"), (np.float64, "64")):
            fc = L.frame_costs(X.frames[path[:, 0]].astype(dt), Y.frames[path[:, 1]].astype(dt))
            assert fc.dtype == dt and np.array_equal(fc, c[f"fc{tag}"])


def test_path_costs_batch_equals_single_calls():
    """cfg4-scale scoring: many long paths in one device call."""
    pairs = [bench.chroma_pair(3000 + 400 * q, 2800 + 300 * q, 12, seed=40 + q) for q in range(6)]
    res = L.align_batch(pairs, precision=32)
    trip = [(X, Y, r.path) for (X, Y), r in zip(pairs, res)]
    many = L.path_costs(trip, dtype=np.float32)
    assert many == [r.cost for r in res]
    assert many == [O.path_cost(X, Y, p, precision=32) for X, Y, p in trip]
    assert L.path_costs(trip, dtype=np.float64) == [O.path_cost(X, Y, p, precision=64) for X, Y, p in trip]


def test_fastdtw_mrmsdtw_at_scale_vs_exact():
    """100k-frame pair: fastdtw (radius 30) and mrmsdtw (1e7 cells) run end to
    end on the device, return valid paths, never beat the exact cost, and
    their discrepancy reports against the exact path are well formed."""
    X, Y = bench.chroma_pair(100000, 90000, 12, seed=77)
    # fp64: the exact optimum bounds every path's cost (up to the summation
    # order of the divide-and-conquer pivots, hence the 1e-12 slack)
    ex = L.linmdtw(X, Y, precision=64)
    for r in (L.fastdtw(X, Y, radius=30, precision=64), L.mrmsdtw(X, Y, max_cells=10 ** 7, precision=64)):
        assert L.validate_path(r.path, 100000, 90000) == []
        assert r.cost >= ex.cost * (1 - 1e-12)
        assert r.cost == L.path_cost(X, Y, r.path, dtype=np.float64)
        rep = L.discrepancy(r.path, ex.path)
        assert rep.errors.shape == (2 * len(r.path),) and (rep.errors >= 0).all()
