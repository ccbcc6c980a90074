"""Parity of the CUDA path (through the C ABI) with the reference golden vectors
and with the CPU oracle, bit-exact: integer outputs (paths, indices, counters)
and the float outputs (diagonals, totals, costs) are compared with ==, in
both fp64 and fp32 accumulation (the kernels reproduce the reference's
unfused, correctly rounded arithmetic, so no tolerance is needed)."""
import numpy as np
import pytest

import bench
import paper_2008_02734_b200 as L
from golden_io import cases, tie_rule, trace_from
from oracle import oracle as O

pytestmark = pytest.mark.gpu

PERMS = [("diag", "left", "up"), ("left", "diag", "up"), ("up", "left", "diag"),
         ("diag", "up", "left"), ("left", "up", "diag"), ("up", "diag", "left")]


def rnd(M, d, seed, kind="gauss"):
    rng = np.random.default_rng(seed)
    if kind == "ties":
        return rng.integers(0, 3, size=(M, d)).astype(np.float32)
    if kind == "walk":
        return (np.cumsum(rng.standard_normal((M, d)), 0) / np.sqrt(M)).astype(np.float32)
    return rng.standard_normal((M, d)).astype(np.float32)


def assert_same_result(r, o):
    assert r.cost == o["cost"]
    assert np.array_equal(r.path, o["path"])
    assert r.cells_processed == o["cells_processed"]
    assert r.peak_diag_values == o["peak_diag_values"]
    assert r.peak_table_cells == o["peak_table_cells"]
    assert list(r.pivot_trace) == list(o["pivot_trace"])


# ------------------------------------------------------------ golden vectors
def test_diag_dtw_golden():
    for case in cases("diag_dtw"):
        b = L.diag_dtw(case["X"], case["Y"], int(case["kstop"]),
                       "reverse" if int(case["reverse"]) else "forward", precision=int(case["prec"]))
        for s in range(3):
            assert np.array_equal(b.d[s], case[f"d{s}"]), (s, case["X"].shape, case["Y"].shape)
            assert np.array_equal(b.c[s], case[f"c{s}"])
        assert b.cells_processed == int(case["cells"])
        assert b.peak_values == int(case["peak"])


def test_dtw_full_golden():
    for case in cases("dtw_full"):
        r = L.dtw_full(case["X"], case["Y"], tie_rule=tie_rule(case["tie"]), precision=int(case["prec"]))
        assert r.cost == float(case["cost"])
        assert np.array_equal(r.path, case["path"])
        if "table" in case:
            assert np.array_equal(L.accumulated_cost_table(case["X"], case["Y"], precision=int(case["prec"])),
                                  case["table"])


def test_find_pivot_golden():
    for case in cases("find_pivot"):
        p = L.find_pivot(case["X"], case["Y"], precision=int(case["prec"]),
                         pivot_tie_rule="highest" if int(case["highest"]) else "lowest")
        assert (p.i, p.j, p.diagonal_k) == (int(case["i"]), int(case["j"]), int(case["k"]))
        assert p.total_at_pivot == float(case["total"])


def test_linmdtw_golden():
    for case in cases("linmdtw"):
        r = L.linmdtw(case["X"], case["Y"], min_dim=int(case["min_dim"]), precision=int(case["prec"]),
                      tie_rule=tie_rule(case["tie"]),
                      pivot_tie_rule="highest" if int(case["highest"]) else "lowest")
        assert r.cost == float(case["cost"])
        assert np.array_equal(r.path, case["path"])
        assert r.cells_processed == int(case["cells"])
        assert r.peak_diag_values == int(case["peak_diag"])
        assert r.peak_table_cells == int(case["peak_table"])
        assert list(r.pivot_trace) == trace_from(case)
        assert r.cells_budget == 2 * case["X"].shape[0] * case["Y"].shape[0]
        assert r.algorithm == "linmdtw"


# --------------------------------------------------- oracle, random shapes
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 12, 16, 48])
def test_diag_dtw_random_vs_oracle(prec, d):
    rng = np.random.default_rng(1000 * d + prec)
    for trial in range(6):
        M, N = (int(v) for v in rng.integers(2, 1500, size=2))
        kind = ("gauss", "ties", "walk")[trial % 3]
        X, Y = rnd(M, d, trial, kind), rnd(N, d, trial + 50, kind)
        kstop = int(rng.integers(2, M + N - 1))
        for direction in ("forward", "reverse"):
            b = L.diag_dtw(X, Y, kstop, direction, precision=prec)
            od, oc, cells = O.half_pass(X, Y, kstop, direction, prec)
            for s in range(3):
                assert np.array_equal(b.d[s], od[s]), (M, N, kstop, direction, s)
                assert np.array_equal(b.c[s], oc[s])
            assert b.cells_processed == cells


@pytest.mark.parametrize("prec", [64, 32])
def test_diag_dtw_every_kstop_small(prec):
    X, Y = rnd(37, 3, 1), rnd(70, 3, 2)
    D, _ = O.fill(X, Y, precision=prec)
    M, N = 37, 70
    for kstop in range(2, M + N - 1):
        b = L.diag_dtw(X, Y, kstop, precision=prec)
        for slot in range(3):
            k = b.diagonal_index(slot)
            i, j = L.diag_cells(k, M, N)
            assert np.array_equal(b.d[slot], D[i, j]), (kstop, slot)


@pytest.mark.parametrize("prec", [64, 32])
def test_dtw_full_random_vs_oracle(prec):
    rng = np.random.default_rng(prec)
    for trial in range(24):
        M, N = (int(v) for v in rng.integers(1, 700, size=2))
        d = int(rng.choice([1, 2, 3, 12, 48]))
        kind = ("gauss", "ties", "walk")[trial % 3]
        X, Y = rnd(M, d, trial, kind), rnd(N, d, trial + 9, kind)
        tie = PERMS[trial % 6]
        r = L.dtw_full(X, Y, tie_rule=tie, precision=prec)
        c, p = O.dtw_full(X, Y, tie, prec)
        assert r.cost == c
        assert np.array_equal(r.path, p), (M, N, d, tie)


@pytest.mark.parametrize("prec", [64, 32])
def test_accumulated_table_vs_oracle(prec):
    for M, N, d in [(1, 1, 1), (1, 50, 2), (50, 1, 2), (65, 64, 3), (200, 333, 12)]:
        X, Y = rnd(M, d, M), rnd(N, d, N + 1)
        D, _ = O.fill(X, Y, precision=prec)
        assert np.array_equal(L.accumulated_cost_table(X, Y, precision=prec), D)


@pytest.mark.parametrize("prec", [64, 32])
def test_find_pivot_random_vs_oracle(prec):
    rng = np.random.default_rng(7 + prec)
    for trial in range(30):
        M, N = (int(v) for v in rng.integers(2, 2000, size=2))
        if M + N - 2 < 2:
            continue
        d = int(rng.choice([1, 2, 12]))
        kind = ("gauss", "ties", "walk")[trial % 3]
        X, Y = rnd(M, d, trial, kind), rnd(N, d, trial + 3, kind)
        for rule in ("lowest", "highest"):
            p = L.find_pivot(X, Y, precision=prec, pivot_tie_rule=rule)
            o = O.find_pivot(X, Y, prec, rule)
            assert (p.i, p.j, p.diagonal_k, p.total_at_pivot) == (o["i"], o["j"], o["diagonal_k"],
                                                                 o["total_at_pivot"]), (M, N, rule)


@pytest.mark.parametrize("prec", [64, 32])
def test_linmdtw_random_vs_oracle(prec):
    rng = np.random.default_rng(31 + prec)
    for trial in range(16):
        M, N = (int(v) for v in rng.integers(1, 2500, size=2))
        d = int(rng.choice([1, 2, 4, 12]))
        md = int(rng.choice([2, 3, 16, 100, 500]))
        kind = ("gauss", "ties", "walk")[trial % 3]
        X, Y = rnd(M, d, trial, kind), rnd(N, d, trial + 1, kind)
        tie = PERMS[trial % 6]
        rule = ("lowest", "highest")[trial % 2]
        r = L.linmdtw(X, Y, min_dim=md, precision=prec, tie_rule=tie, pivot_tie_rule=rule)
        o = O.linmdtw(X, Y, min_dim=md, precision=prec, tie_rule=tie, pivot_tie_rule=rule, nthreads=8)
        assert_same_result(r, o)


def test_edge_shapes():
    for M, N in [(1, 1), (1, 7), (7, 1), (2, 2), (2, 3), (3, 2), (1, 4), (4, 1), (65, 1), (1, 129)]:
        for prec in (32, 64):
            X, Y = rnd(M, 2, M), rnd(N, 2, N + 7)
            r = L.linmdtw(X, Y, min_dim=2, precision=prec)
            o = O.linmdtw(X, Y, min_dim=2, precision=prec)
            assert_same_result(r, o)
            r = L.dtw_full(X, Y, precision=prec)
            c, p = O.dtw_full(X, Y, precision=prec)
            assert r.cost == c and np.array_equal(r.path, p)


def test_constant_series_all_ties():
    X = np.ones((300, 4), np.float32)
    Y = np.ones((257, 4), np.float32)
    for rule in ("lowest", "highest"):
        for tie in PERMS[:3]:
            r = L.linmdtw(X, Y, min_dim=8, tie_rule=tie, pivot_tie_rule=rule)
            o = O.linmdtw(X, Y, min_dim=8, tie_rule=tie, pivot_tie_rule=rule)
            assert_same_result(r, o)
            assert r.cost == 0.0


def test_align_batch_equals_single_calls():
    rng = np.random.default_rng(5)
    pairs = []
    for q in range(9):
        M, N = (int(v) for v in rng.integers(1, 1200, size=2))
        pairs.append((rnd(M, 12, q, "walk"), rnd(N, 12, q + 100, "walk")))
    for prec in (32, 64):
        batch = L.align_batch(pairs, min_dim=64, precision=prec)
        for (X, Y), r in zip(pairs, batch):
            s = L.linmdtw(X, Y, min_dim=64, precision=prec)
            assert r.cost == s.cost and np.array_equal(r.path, s.path)
            assert r.cells_processed == s.cells_processed and r.pivot_trace == s.pivot_trace


def test_progress_contract():
    X, Y = rnd(150, 2, 8), rnd(170, 2, 9)
    seen = []
    r = L.linmdtw(X, Y, min_dim=16, progress=lambda done, budget: seen.append((done, budget)))
    done = [d for d, _ in seen]
    assert done == sorted(done)
    assert seen[-1] == (r.cells_processed, 2 * 150 * 170)
    gaps = np.diff(done)
    assert np.all(gaps <= max(1, 2 * 150 * 170 // 100) + 6 * min(150, 170))


def test_on_cells_accumulates_to_total():
    X, Y = rnd(64, 2, 0), rnd(59, 2, 1)
    seen = []
    b = L.diag_dtw(X, Y, kstop=100, on_cells=seen.append)
    assert sum(seen) == b.cells_processed and all(n > 0 for n in seen)


# ----------------------------------------------- larger sizes, properties
@pytest.mark.parametrize("prec", [32, 64])
def test_medium_chroma_vs_oracle(prec):
    """cfg2-style generator at 4k x 3.5k: full result equality with the oracle."""
    import bench
    X, Y = bench.chroma_pair(4000, 3500, 12, seed=2)
    r = L.linmdtw(X, Y, precision=prec)
    o = O.linmdtw(X, Y, precision=prec, nthreads=16)
    assert_same_result(r, o)


def test_linmdtw_matches_full_table_dtw_at_scale():
    """Size-independent property at 20k x 18k (fp64): the divide-and-conquer path
    and cost equal the brute-force DTW's on tie-free inputs."""
    import bench
    X, Y = bench.chroma_pair(20000, 18000, 12, seed=11)
    r = L.linmdtw(X, Y, precision=64)
    f = L.dtw_full(X, Y, precision=64)
    assert L.validate_path(r.path, 20000, 18000) == []
    assert np.array_equal(r.path, f.path)
    assert r.cost == f.cost
    assert 1.8 < r.cells_processed / (20000 * 18000) <= 2.0 + 1e-3


def test_cfg5_shape_skinny_fp64_vs_oracle():
    """BASELINE cfg5's generator (random-walk latent, d=48, fp64, 10:1 aspect)
    at 40k x 4k: path, cost, counters and pivot trace equal the oracle's;
    the lopsided tree ends in skinny leaves."""
    X, Y = bench.latent_pair(40000, 4000, 48, seed=5)
    r = L.linmdtw(X, Y, precision=64)
    o = O.linmdtw(X, Y, precision=64, nthreads=16)
    assert_same_result(r, o)
    assert max(t["M"] for t in r.pivot_trace) == 40000 and r.peak_table_cells > 0


def test_cfg4_shape_batch_vs_oracle():
    """BASELINE cfg4's shape (a batch of pairs with random lengths, chroma d=12,
    fp32) scaled to lengths in [500, 3000]: every result of the fused batch
    equals the oracle's single alignment."""
    rng = np.random.default_rng(4)
    MN = rng.integers(500, 3001, size=(12, 2))
    pairs = [bench.chroma_pair(int(m), int(n), 12, seed=1000 + q) for q, (m, n) in enumerate(MN)]
    batch = L.align_batch(pairs, precision=32)
    for (X, Y), r in zip(pairs, batch):
        assert_same_result(r, O.linmdtw(X, Y, precision=32, nthreads=16))


def _dist_gpu_worker(rank, world, port, cases, q):
    import os
    import torch.distributed as dist
    from paper_2008_02734_b200.distributed import linmdtw_distributed
    # shards in different processes share the GPU by time slicing: allow long waits
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LMDTW_WATCHDOG_S="120")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for M, N, d, seed, prec, min_dim in cases:
            X, Y = bench.chroma_pair(M, N, d, seed=seed)
            r = linmdtw_distributed(X, Y, min_dim=min_dim, precision=prec)
            out.append((r.cost, r.path, r.cells_processed, r.peak_diag_values, r.peak_table_cells,
                        list(r.pivot_trace)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_device_engine_equals_single_gpu(world):
    """Ranks (gloo) sharing cuda:0 through the C ABI: top-level half passes
    split across ranks (with 3 ranks one half pass is cut into two strip
    shards whose handoff crosses processes through a CUDA IPC buffer), pivots
    combined on the host, leaves sharded; the result equals the single-GPU
    engine's bit for bit."""
    import socket
    import torch.multiprocessing as mp
    cases = [(3000, 2600, 12, 7, 32, 500), (2200, 1800, 5, 8, 64, 300)]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_gpu_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (M, N, d, seed, prec, min_dim) in enumerate(cases):
        X, Y = bench.chroma_pair(M, N, d, seed=seed)
        ref = L.linmdtw(X, Y, min_dim=min_dim, precision=prec)
        for rank in range(world):
            cost, path, cells, pkd, pkt, trace = res[rank][ci]
            assert cost == ref.cost and np.array_equal(path, ref.path)
            assert cells == ref.cells_processed and pkd == ref.peak_diag_values and pkt == ref.peak_table_cells
            assert trace == list(ref.pivot_trace)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("reverse", [0, 1])
def test_strip_sharded_half_pass_equals_unsharded(prec, reverse):
    """The strip-sharding mechanism of the multi-GPU layout, on one GPU: a half
    pass split into 2-4 contiguous strip ranges, each a separate persistent
    kernel on its own stream and buffers running concurrently, the first strip
    of every range reading the previous range's handoff buffer with
    system-scope loads.  The merged last three diagonals equal the unsharded
    pass bit for bit."""
    import ctypes as C
    from paper_2008_02734_b200 import _capi
    lib = _capi.load()
    dt = np.float32 if prec == 32 else np.float64
    for (M, N, d, kfrac, seed) in [(1500, 5200, 12, 0.5, 1), (2100, 4300, 3, 0.8, 2), (900, 2500, 12, 1.0, 3)]:
        X, Y = bench.chroma_pair(M, N, d, seed=seed)
        kstop = max(2, min(M + N - 2, int(kfrac * (M + N - 2))))
        lens = [L.diag_length(kstop - 2 + s, M, N) for s in range(3)]
        ref = L.diag_dtw(X, Y, kstop, "reverse" if reverse else "forward", precision=prec)
        for ns in (2, 3, 4):
            od = [np.full(max(n, 1), np.nan, dt) for n in lens]
            oc = [np.full(max(n, 1), np.nan, dt) for n in lens]
            pd = (C.c_void_p * 3)(*[o.ctypes.data for o in od])
            pc = (C.c_void_p * 3)(*[o.ctypes.data for o in oc])
            _capi.check(lib.lmdtw_debug_sharded_half_pass(
                0, _capi.ptr(X), C.c_int64(M), _capi.ptr(Y), C.c_int64(N), d, C.c_int64(kstop), reverse, prec, ns,
                pd, pc))
            for s in range(3):
                assert np.array_equal(od[s][:lens[s]], ref.d[s]), (M, N, ns, s)
                assert np.array_equal(oc[s][:lens[s]], ref.c[s]), (M, N, ns, s)


def test_cfg3_full_size_linmdtw_equals_full_table_dtw_fp64():
    """BASELINE cfg3 at full size (100k x 100k, d=12, the bench's inputs), fp64:
    the linear-memory path and cost equal the brute-force DTW's (full table
    of 2-bit backpointers on the device, 2.5 GB) -- the reference's own
    acceptance property (test_divide.py:80-86) at the headline shape."""
    X, Y = bench.make_inputs("cfg3")[0]
    r = L.linmdtw(X, Y, precision=64)
    f = L.dtw_full(X, Y, precision=64)
    assert np.array_equal(r.path, f.path)
    assert r.cost == f.cost
    assert r.cells_processed == 19910735310 or 1.99 < r.cells_processed / 1e10 < 2.0


def test_cfg3_full_size_fp32_equals_oracle():
    """The bench workload itself (cfg3, fp32): path, cost, cells_processed, peak
    counters and the 255-entry pivot trace equal the C oracle's (the reference
    algorithm restated, run on all host cores, ~1 min)."""
    X, Y = bench.make_inputs("cfg3")[0]
    r = L.linmdtw(X, Y, precision=32)
    o = O.linmdtw(X, Y, precision=32, nthreads=O.num_threads())
    assert_same_result(r, o)
    assert len(r.pivot_trace) == 255
