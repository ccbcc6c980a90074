"""Full-size parity at every BASELINE.json config against the CPU oracle (the
reference algorithm restated in C, pinned to the reference's golden vectors),
plus the reference's acceptance sweep replayed on the GPU.  Bit-exact, no
tolerances: path, cost, cells_processed, peak counters and the pre-order
pivot trace.  The oracle runs on all host cores (its long diagonals are
split into tasks; results never depend on the thread count)."""
import numpy as np
import pytest

import bench
import paper_2008_02734_b200 as L
from oracle import oracle as O

pytestmark = pytest.mark.gpu

NT = O.num_threads()


def assert_same_result(r, o):
    assert r.cost == o["cost"]
    assert np.array_equal(r.path, o["path"])
    assert r.cells_processed == o["cells_processed"]
    assert r.peak_diag_values == o["peak_diag_values"]
    assert r.peak_table_cells == o["peak_table_cells"]
    assert list(r.pivot_trace) == list(o["pivot_trace"])


def test_acceptance_c1_sweep_gpu():
    """Reference acceptance criterion 1 (test_acceptance.py:40-74) on the GPU:
    2,178 tiny instances (dims 1 and 4, M, N in 2..12) at min_dim=2; results
    equal the reference's linmdtw (golden, fp64 and fp32) and the fp64 cost
    equals the OptimalPathDag-certified minimum."""
    from golden_io import acceptance_c1
    for rec in acceptance_c1():
        for prec in (32, 64):
            r = L.linmdtw(rec["X"], rec["Y"], min_dim=2, precision=prec)
            g = rec[prec]
            assert r.cost == g["cost"]
            assert np.array_equal(r.path, g["path"])
            assert list(r.pivot_trace) == g["trace"]
        assert rec[64]["cost"] == rec["dag_cost"]


@pytest.mark.parametrize("prec", [32, 64])
def test_cfg2_full_size_vs_oracle(prec):
    """BASELINE cfg2 (20k x 20k, d=12 chroma, seed 2) at its real shape."""
    X, Y = bench.make_inputs("cfg2")[0]
    r = L.linmdtw(X, Y, precision=prec)
    o = O.linmdtw(X, Y, precision=prec, nthreads=NT)
    assert_same_result(r, o)
    assert r.cells_processed == 793265172 or prec == 64


def test_cfg3_full_size_fp64_vs_oracle():
    """BASELINE cfg3 (100k x 100k, d=12) in fp64: equal to the oracle field by
    field (the fp32 run is test_gpu_parity.test_cfg3_full_size_fp32_equals_oracle)."""
    X, Y = bench.make_inputs("cfg3")[0]
    r = L.linmdtw(X, Y, precision=64)
    o = O.linmdtw(X, Y, precision=64, nthreads=NT)
    assert_same_result(r, o)
    assert len(r.pivot_trace) == 255


def test_cfg5_full_size_vs_oracle():
    """BASELINE cfg5 -- the path-identical check: M=200,000, N=20,000, d=48,
    fp64 (correlated latent walk, seed 5)."""
    X, Y = bench.make_inputs("cfg5")[0]
    r = L.linmdtw(X, Y, precision=64)
    o = O.linmdtw(X, Y, precision=64, nthreads=NT)
    assert_same_result(r, o)


def test_cfg5_independent_walks_skinny_leaves_vs_oracle():
    """cfg5's shape with INDEPENDENT random walks (the survey's measurement,
    SURVEY.md 8(d) cfg5): a lopsided recursion whose leaves are long and
    skinny (tens of thousands of rows by a few dozen columns); equal to the
    oracle, and the skinny leaves really occur."""
    rng = np.random.default_rng(55)
    X = (np.cumsum(rng.standard_normal((200000, 48)), 0) / np.sqrt(200000)).astype(np.float32)
    Y = (np.cumsum(rng.standard_normal((20000, 48)), 0) / np.sqrt(20000)).astype(np.float32)
    r = L.linmdtw(X, Y, precision=64)
    o = O.linmdtw(X, Y, precision=64, nthreads=NT)
    assert_same_result(r, o)
    assert r.peak_table_cells >= 10000 * 2  # a leaf of >= 10k rows by >= 2 columns at least


def test_cfg4_subsample_full_lengths_vs_oracle():
    """BASELINE cfg4 at full lengths: the first 32 pairs of the 256-pair batch
    (M, N in [5k, 30k]) aligned as one fused batch; every result equals the
    oracle's single alignment."""
    pairs = bench.make_inputs("cfg4")[:32]
    batch = L.align_batch(pairs, precision=32)
    for (X, Y), r in zip(pairs, batch):
        assert_same_result(r, O.linmdtw(X, Y, precision=32, nthreads=NT))


@pytest.mark.parametrize("shape", [(110000, 32), (32, 110000)])
def test_dtw_full_skinny_fp64_vs_oracle(shape):
    """Leaf solver on the survey's worst cfg5 leaf shape (109,968 x 32, SURVEY
    8(a) a19) and its transpose, fp64: cost and path equal the oracle's."""
    M, N = shape
    rng = np.random.default_rng(M + 7 * N)
    X = (np.cumsum(rng.standard_normal((M, 48)), 0) / np.sqrt(M)).astype(np.float32)
    Y = (np.cumsum(rng.standard_normal((N, 48)), 0) / np.sqrt(N)).astype(np.float32)
    f = L.dtw_full(X, Y, precision=64)
    c, p = O.dtw_full(X, Y, precision=64)
    assert f.cost == c
    assert np.array_equal(f.path, p)


@pytest.mark.parametrize("prec", [32, 64])
def test_d100_audio_features_vs_oracle(prec):
    """The reference extractor's feature width (mfcc-mod / DLNC0: d = 100,
    extractor features.py:62-65) at 8k x 7k on the WIDE (dimension-blocked)
    kernels: equal to the oracle in both precisions."""
    X, Y = bench.latent_pair(8000, 7000, 100, seed=100)
    r = L.linmdtw(X, Y, precision=prec)
    o = O.linmdtw(X, Y, precision=prec, nthreads=NT)
    assert_same_result(r, o)
