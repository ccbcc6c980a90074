"""Pin the CPU oracle (oracle/lmdtw_oracle.c) against golden vectors produced by
the real reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from golden_io import cases, tie_rule, trace_from
from oracle import oracle as O


@pytest.mark.parametrize("case", cases("diag_dtw"), ids=lambda c: f"M{c['X'].shape[0]}N{c['Y'].shape[0]}")
def test_half_pass_matches_reference(case):
    d, c, cells = O.half_pass(case["X"], case["Y"], int(case["kstop"]),
                              "reverse" if int(case["reverse"]) else "forward", int(case["prec"]))
    for s in range(3):
        assert np.array_equal(d[s], case[f"d{s}"])
        assert np.array_equal(c[s], case[f"c{s}"])
    assert cells == int(case["cells"])
    assert O.peak_retained_values(int(case["kstop"]), case["X"].shape[0], case["Y"].shape[0]) == int(case["peak"])


def test_dtw_full_matches_reference():
    for case in cases("dtw_full"):
        cost, path = O.dtw_full(case["X"], case["Y"], tie_rule(case["tie"]), int(case["prec"]))
        assert cost == float(case["cost"])
        assert np.array_equal(path, case["path"])
        if "table" in case:
            D, _ = O.fill(case["X"], case["Y"], tie_rule(case["tie"]), int(case["prec"]))
            assert np.array_equal(D, case["table"])


def test_find_pivot_matches_reference():
    for case in cases("find_pivot"):
        p = O.find_pivot(case["X"], case["Y"], int(case["prec"]),
                         "highest" if int(case["highest"]) else "lowest")
        assert (p["i"], p["j"], p["diagonal_k"]) == (int(case["i"]), int(case["j"]), int(case["k"]))
        assert p["total_at_pivot"] == float(case["total"])


@pytest.mark.parametrize("nthreads", [1, 4])
def test_linmdtw_matches_reference(nthreads):
    for case in cases("linmdtw"):
        r = O.linmdtw(case["X"], case["Y"], min_dim=int(case["min_dim"]), precision=int(case["prec"]),
                      tie_rule=tie_rule(case["tie"]),
                      pivot_tie_rule="highest" if int(case["highest"]) else "lowest", nthreads=nthreads)
        assert r["cost"] == float(case["cost"])
        assert np.array_equal(r["path"], case["path"])
        assert r["cells_processed"] == int(case["cells"])
        assert r["peak_diag_values"] == int(case["peak_diag"])
        assert r["peak_table_cells"] == int(case["peak_table"])
        assert list(r["pivot_trace"]) == trace_from(case)


def test_path_cost_matches_reference():
    for case in cases("linmdtw"):
        assert O.path_cost(case["X"], case["Y"], case["path"], int(case["prec"])) == float(case["cost"])


def test_cfg1_golden_values():
    """SURVEY §8(d) cfg1 golden values, recorded from the reference."""
    c64, c32 = cases("linmdtw")[:2]
    assert float(c64["cost"]) == 11.1431643162049
    assert float(c32["cost"]) == 11.14316463470459
    assert int(c64["cells"]) == 1501687 and len(c64["path"]) == 1073


def test_acceptance_c1_sweep_oracle():
    """Reference acceptance criterion 1 (test_acceptance.py:40-74): 2,178 tiny
    instances at min_dim=2.  The oracle's linmdtw equals the reference's result
    (cost, path, pivot trace) in fp64 and fp32, and the fp64 cost equals the
    OptimalPathDag-certified minimum the reference checks against."""
    from golden_io import acceptance_c1
    for rec in acceptance_c1():
        assert rec[64]["cost"] == rec["dag_cost"]
        for prec in (32, 64):
            o = O.linmdtw(rec["X"], rec["Y"], min_dim=2, precision=prec)
            assert o["cost"] == rec[prec]["cost"]
            assert np.array_equal(o["path"], rec[prec]["path"])
            assert list(o["pivot_trace"]) == rec[prec]["trace"]


def test_window_dtw_matches_reference():
    """Oracle constrained_dtw (approx.py:180-220) against the reference's
    results on windows from window_from_path / expand_window / Window.full."""
    from golden_io import approx_cases
    for c in approx_cases("cw"):
        cost, path, cells = O.window_dtw(c["X"], c["Y"], c["lo"], c["hi"], tie_rule(c["tie"]), int(c["prec"]))
        assert cost == float(c["cost"])
        assert np.array_equal(path, c["path"])
        assert cells == int(c["cells"])
