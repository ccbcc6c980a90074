"""Host-side API behaviour that precedes any device call (validation and
types), ported from the reference's unit tests.  CPU only."""
import numpy as np
import pytest

import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import InvalidInputError


def series(v):
    return L.FeatureSeries(np.asarray(v, np.float32).reshape(-1, 1), 100.0)


class TestIndexing:  # reference tests/test_diagonal.py:12-45
    def test_lengths(self):
        assert L.diag_length(0, 3, 3) == 1
        assert L.diag_length(2, 3, 3) == 3
        assert L.diag_length(3, 2, 3) == 1

    def test_length_sums_to_grid(self):
        for M, N in [(1, 1), (1, 7), (4, 3), (9, 2)]:
            assert sum(L.diag_length(k, M, N) for k in range(M + N - 1)) == M * N

    def test_out_of_range(self):
        with pytest.raises(InvalidInputError):
            L.diag_length(5, 3, 3)

    def test_grid_convention_anchors(self):
        assert L.diag_to_grid(2, 0, 3, 3) == (2, 0)
        assert L.diag_to_grid(2, 2, 3, 3) == (0, 2)
        assert L.diag_to_grid(3, 0, 2, 3) == (1, 2)

    def test_bijection(self):
        M, N = 4, 6
        seen = set()
        for k in range(M + N - 1):
            for idx in range(L.diag_length(k, M, N)):
                i, j = L.diag_to_grid(k, idx, M, N)
                assert i + j == k and 0 <= i < M and 0 <= j < N
                seen.add((i, j))
        assert len(seen) == M * N

    def test_diag_cells_matches_scalar(self):
        for k in range(8):
            i, j = L.diag_cells(k, 4, 5)
            assert [tuple(x) for x in zip(i, j)] == [L.diag_to_grid(k, idx, 4, 5)
                                                     for idx in range(L.diag_length(k, 4, 5))]

    def test_peak_values_bound(self):
        for M, N in [(2, 2), (5, 9), (50, 50), (120, 40)]:
            assert L.peak_retained_values(M + N - 2, M, N) <= 6 * min(M, N)


class TestValidation:
    def test_kstop_validation(self):
        X = np.zeros((4, 1), np.float32)
        for bad in (1, 7):
            with pytest.raises(InvalidInputError):
                L.diag_dtw(X, X, kstop=bad)
        with pytest.raises(InvalidInputError):
            L.diag_dtw(series([0]), series([0]), kstop=2)

    def test_direction(self):
        X = np.zeros((4, 1), np.float32)
        with pytest.raises(InvalidInputError):
            L.diag_dtw(X, X, kstop=3, direction="sideways")

    def test_find_pivot_too_small(self):
        with pytest.raises(InvalidInputError):
            L.find_pivot(series([0]), series([1]))

    def test_config(self):
        with pytest.raises(InvalidInputError):
            L.LinMdtwConfig(min_dim=1)
        with pytest.raises(InvalidInputError):
            L.LinMdtwConfig(pivot_tie_rule="middle")
        X = np.zeros((10, 1), np.float32)
        with pytest.raises(InvalidInputError):
            L.linmdtw(X, X, config=L.LinMdtwConfig(), min_dim=4)

    def test_cost_kind_and_dims(self):
        X = np.zeros((5, 2), np.float32)
        Y = np.zeros((5, 3), np.float32)
        with pytest.raises(InvalidInputError):
            L.linmdtw(X, X, cost="cosine")
        with pytest.raises(InvalidInputError):
            L.linmdtw(X, Y)
        with pytest.raises(InvalidInputError):
            L.dtw_full(X, Y)

    def test_bad_tie_rule_and_precision(self):
        X = np.zeros((5, 2), np.float32)
        with pytest.raises(InvalidInputError):
            L.dtw_full(X, X, tie_rule=("diag", "diag", "up"))
        with pytest.raises(InvalidInputError):
            L.dtw_full(X, X, precision=16)
        with pytest.raises(InvalidInputError):
            L.linmdtw(X, X, precision="half")

    def test_feature_series(self):
        with pytest.raises(InvalidInputError):
            L.FeatureSeries(np.array([[np.nan]]))
        with pytest.raises(InvalidInputError):
            L.FeatureSeries(np.zeros((0, 2)))
        s = L.as_series([1, 2, 3])
        assert s.frames.shape == (3, 1) and s.frames.dtype == np.float32
        assert not s.frames.flags.writeable
        assert np.array_equal(s.reversed().frames[:, 0], [3, 2, 1])
        assert np.array_equal(s.view(1, 3).frames[:, 0], [2, 3])
        with pytest.raises(InvalidInputError):
            s.view(2, 2)

    def test_precision_dtype(self):
        assert L.precision_dtype(32) == np.float32
        assert L.precision_dtype("float64") == np.float64
        with pytest.raises(InvalidInputError):
            L.precision_dtype(8)

    def test_validate_path(self):
        assert L.validate_path([(0, 0), (1, 1)], 2, 2) == []
        v = L.validate_path([(0, 0), (0, 0), (1, 1)], 2, 2)
        assert any(x.startswith("illegal-step") for x in v)
        v = L.validate_path([(0, 0), (1, 2), (1, 1)], 2, 2)
        assert any(x.startswith("index-out-of-range") for x in v)
        with pytest.raises(L.PathValidationError):
            L.require_valid_path([(0, 1), (1, 1)], 2, 2)

    def test_tie_codes(self):
        assert list(L.tie_codes(L.TIE_DIAG_FIRST)) == [2, 0, 1]
        assert list(L.tie_codes(L.TIE_LEFT_FIRST)) == [0, 2, 1]

    def test_host_backtrace_helper(self):
        P = np.array([[3, 0, 0], [1, 2, 2]], np.uint8)
        assert [tuple(p) for p in L.backtrace(P)] == [(0, 0), (0, 1), (1, 2)]
        with pytest.raises(RuntimeError):
            L.backtrace(np.array([[3, 3], [3, 3]], np.uint8))
