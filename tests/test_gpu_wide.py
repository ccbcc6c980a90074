"""Any feature dimension (the reference accepts every d >= 1; its
own extractor emits d = 100, extractor/src/lmdtw_extract/features.py:62-65).
Rows longer than the register-resident kernels take (d > 64 in fp32, d > 48
in fp64) run the dimension-blocked WIDE kernels; these tests compare them
with the oracle bit for bit, through the C ABI."""
import numpy as np
import pytest

import bench
import paper_2008_02734_b200 as L
from oracle import oracle as O
from test_gpu_parity import PERMS, assert_same_result, rnd

pytestmark = pytest.mark.gpu

WIDE_DIMS = [49, 65, 100, 128, 256, 300]


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("d", WIDE_DIMS)
def test_wide_diag_dtw_vs_oracle(prec, d):
    rng = np.random.default_rng(77 * d + prec)
    for trial in range(3):
        M, N = (int(v) for v in rng.integers(2, 900, size=2))
        kind = ("gauss", "ties", "walk")[trial % 3]
        X, Y = rnd(M, d, trial, kind), rnd(N, d, trial + 50, kind)
        kstop = int(rng.integers(2, M + N - 1))
        for direction in ("forward", "reverse"):
            b = L.diag_dtw(X, Y, kstop, direction, precision=prec)
            od, oc, cells = O.half_pass(X, Y, kstop, direction, prec)
            for s in range(3):
                assert np.array_equal(b.d[s], od[s]), (d, M, N, kstop, direction, s)
                assert np.array_equal(b.c[s], oc[s])
            assert b.cells_processed == cells


@pytest.mark.parametrize("prec", [64, 32])
def test_wide_dtw_full_vs_oracle(prec):
    rng = np.random.default_rng(5 + prec)
    for trial, d in enumerate([65, 100, 128, 100, 256, 97]):
        M, N = (int(v) for v in rng.integers(1, 600, size=2))
        kind = ("gauss", "ties", "walk")[trial % 3]
        X, Y = rnd(M, d, trial, kind), rnd(N, d, trial + 9, kind)
        tie = PERMS[trial % 6]
        r = L.dtw_full(X, Y, tie_rule=tie, precision=prec)
        c, p = O.dtw_full(X, Y, tie, prec)
        assert r.cost == c
        assert np.array_equal(r.path, p), (M, N, d, tie)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("d", [100, 128])
def test_wide_linmdtw_vs_oracle(prec, d):
    """The reference's audio features (d = 100) through the whole aligner."""
    X, Y = bench.chroma_pair(2600, 2200, d, seed=d)
    r = L.linmdtw(X, Y, min_dim=300, precision=prec)
    o = O.linmdtw(X, Y, min_dim=300, precision=prec, nthreads=O.num_threads())
    assert_same_result(r, o)


def test_wide_find_pivot_vs_oracle():
    for prec in (32, 64):
        for rule in ("lowest", "highest"):
            X, Y = rnd(1300, 100, 1, "ties"), rnd(1100, 100, 2, "ties")
            p = L.find_pivot(X, Y, precision=prec, pivot_tie_rule=rule)
            o = O.find_pivot(X, Y, prec, rule)
            assert (p.i, p.j, p.diagonal_k, p.total_at_pivot) == (o["i"], o["j"], o["diagonal_k"],
                                                                 o["total_at_pivot"])


@pytest.mark.parametrize("prec", [64, 32])
def test_wide_multi_tile_vs_oracle(prec):
    """Passes longer than one 8192-column tile on the WIDE kernels: tile
    boundaries (left-boundary handoff between tiles of a strip), the static
    first round of work items and the cp.async-staged X / Y blocks across
    tiles; a half pass in both directions and a skinny brute-force leaf."""
    d = 100
    X, Y = rnd(700, d, 3, "walk"), rnd(18000, d, 4, "walk")
    kstop = (700 + 18000) // 2
    for direction in ("forward", "reverse"):
        b = L.diag_dtw(X, Y, kstop, direction, precision=prec)
        od, oc, cells = O.half_pass(X, Y, kstop, direction, prec)
        for s in range(3):
            assert np.array_equal(b.d[s], od[s]), (direction, s)
            assert np.array_equal(b.c[s], oc[s])
        assert b.cells_processed == cells
    Xs = X[:40]
    r = L.dtw_full(Xs, Y, tie_rule=PERMS[0], precision=prec)
    c, p = O.dtw_full(Xs, Y, PERMS[0], prec)
    assert r.cost == c
    assert np.array_equal(r.path, p)
