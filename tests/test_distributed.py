"""Multi-rank recursion (paper_2008_02734_b200/distributed.py) on CPU.

The partition and exchange logic runs under torch.distributed with the gloo
backend (world sizes 2 and 3, 127.0.0.1 rendezvous).  The per-rank compute is
a test engine over the C oracle (test infrastructure, never shipped); the
split-point combine and path_cost are the product's host entry points
(lmdtw_pivot_combine, lmdtw_path_cost).  Every rank's result must equal the
single-process oracle linmdtw bit for bit: path, cost, cells_processed, peak
counters and the pre-order pivot trace.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import _capi
from paper_2008_02734_b200.distributed import lpt_assign, linmdtw_distributed
from oracle import oracle as O


class OracleEngine:
    """Test-only per-rank compute: the C oracle on sub-block views."""

    def __init__(self, X, Y, cfg):
        self.X = np.ascontiguousarray(X, np.float32)
        self.Y = np.ascontiguousarray(Y, np.float32)
        self.cfg = cfg
        self.prec = int(cfg.precision)
        self.calls = []

    def pivot_nodes(self, subs):
        out = []
        for i0, j0, m, n in subs:
            self.calls.append(("pivot", m, n))
            p = O.find_pivot(self.X[i0:i0 + m], self.Y[j0:j0 + n], self.prec, self.cfg.pivot_tie_rule)
            out.append((p["i"], p["j"], p["diagonal_k"], p["total_at_pivot"]))
        return out

    def half_pass(self, sub, reverse):
        i0, j0, m, n = sub
        self.calls.append(("half", m, n, reverse))
        K = m + n - 1
        kf = (K + 1) // 2
        kb = kf + 1 if K % 2 == 0 else kf
        d, c, _ = O.half_pass(self.X[i0:i0 + m], self.Y[j0:j0 + n], kb if reverse else kf,
                              "reverse" if reverse else "forward", self.prec)
        return list(d), list(c)

    def combine(self, M, N, fwd_d, fwd_c, bwd_d):
        lib = _capi.load()
        fd = (C.c_void_p * 3)(*[np.ascontiguousarray(a).ctypes.data for a in fwd_d])
        fc = (C.c_void_p * 3)(*[np.ascontiguousarray(a).ctypes.data for a in fwd_c])
        bd = (C.c_void_p * 3)(*[np.ascontiguousarray(a).ctypes.data for a in bwd_d])
        ijk = np.zeros(3, np.int64)
        tot = C.c_double()
        _capi.check(lib.lmdtw_pivot_combine(self.prec, M, N, 1 if self.cfg.pivot_tie_rule == "highest" else 0,
                                            fd, fc, bd, _capi.ptr(ijk), C.byref(tot)))
        return int(ijk[0]), int(ijk[1]), int(ijk[2]), float(tot.value)

    def leaves(self, subs):
        out = []
        for i0, j0, m, n in subs:
            self.calls.append(("leaf", m, n))
            _, p = O.dtw_full(self.X[i0:i0 + m], self.Y[j0:j0 + n], self.cfg.tie_rule, self.prec)
            out.append(p)
        return out

    def path_cost(self, path):
        lib = _capi.load()
        cost = C.c_double()
        p = np.ascontiguousarray(path, np.int64)
        _capi.check(lib.lmdtw_path_cost(_capi.ptr(self.X), self.X.shape[0], _capi.ptr(self.Y), self.Y.shape[0],
                                        self.X.shape[1], _capi.ptr(p), p.shape[0], self.prec, C.byref(cost)))
        return float(cost.value)


def _pair(M, N, d, seed, integer=False):
    rng = np.random.default_rng(seed)
    if integer:  # tie-heavy
        return (rng.integers(0, 3, (M, d)).astype(np.float32), rng.integers(0, 3, (N, d)).astype(np.float32))
    w = np.cumsum(rng.standard_normal((max(M, N), d)), 0).astype(np.float32)
    return w[:M].copy(), (w[:N] + 0.05 * rng.standard_normal((N, d))).astype(np.float32)


CASES = [
    # (M, N, d, seed, integer, min_dim, precision, pivot_tie_rule)
    (300, 260, 3, 1, False, 32, 64, "lowest"),
    (257, 301, 2, 2, False, 16, 32, "lowest"),
    (120, 140, 1, 3, True, 8, 64, "highest"),
    (90, 400, 4, 4, False, 20, 64, "lowest"),
]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for M, N, d, seed, integer, min_dim, prec, rule in CASES:
            X, Y = _pair(M, N, d, seed, integer)
            cfg = L.LinMdtwConfig(min_dim=min_dim, precision=prec, pivot_tie_rule=rule)
            eng = OracleEngine(X, Y, cfg)
            r = linmdtw_distributed(X, Y, config=cfg, engine=eng)
            out.append((r.cost, r.path, r.cells_processed, r.peak_diag_values, r.peak_table_cells,
                        list(r.pivot_trace), eng.calls))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_equals_single_process_oracle(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (M, N, d, seed, integer, min_dim, prec, rule) in enumerate(CASES):
        X, Y = _pair(M, N, d, seed, integer)
        ref = O.linmdtw(X, Y, min_dim=min_dim, precision=prec, pivot_tie_rule=rule)
        calls = []
        for rank in range(world):
            cost, path, cells, pkd, pkt, trace, rcalls = results[rank][ci]
            assert cost == ref["cost"]
            assert np.array_equal(path, ref["path"])
            assert cells == ref["cells_processed"]
            assert pkd == ref["peak_diag_values"] and pkt == ref["peak_table_cells"]
            assert trace == list(ref["pivot_trace"])
            calls += rcalls
        # the work is partitioned, not replicated: every leaf solved exactly once
        nleaf = sum(1 for c in calls if c[0] == "leaf")
        assert nleaf == len(ref["pivot_trace"]) + 1
        # the top node was split into its two half passes on different ranks
        tops = [c for c in calls if c[0] == "half" and c[1] == M and c[2] == N]
        assert sorted(c[3] for c in tops) == [0, 1]


def test_lpt_assign_balances_and_is_deterministic():
    w = [9, 7, 5, 5, 3, 1]
    owner = lpt_assign(w, 3)
    loads = [sum(x for x, o in zip(w, owner) if o == r) for r in range(3)]
    assert sorted(loads) == [10, 10, 10]
    assert lpt_assign(w, 3) == owner
    assert lpt_assign([], 4) == []
    assert set(lpt_assign([1] * 8, 8)) == set(range(8))


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("rule", ["lowest", "highest"])
def test_pivot_combine_matches_oracle_find_pivot(prec, rule):
    """lmdtw_pivot_combine (host) on oracle half passes == oracle find_pivot."""
    rng = np.random.default_rng(7)
    for t in range(25):
        M, N = int(rng.integers(2, 60)), int(rng.integers(2, 60))
        if M + N - 2 < 2:
            continue
        integer = t % 3 == 0
        X, Y = _pair(M, N, 2, 100 + t, integer)
        cfg = L.LinMdtwConfig(min_dim=2, precision=prec, pivot_tie_rule=rule)
        eng = OracleEngine(X, Y, cfg)
        fd, fc = eng.half_pass((0, 0, M, N), 0)
        bd, _ = eng.half_pass((0, 0, M, N), 1)
        i, j, k, tot = eng.combine(M, N, fd, fc, bd)
        ref = O.find_pivot(X, Y, prec, rule)
        assert (i, j, k) == (ref["i"], ref["j"], ref["diagonal_k"]), (M, N, t)
        assert tot == ref["total_at_pivot"]


def test_strip_ranges_and_apportion():
    """Shard planning helpers (host only)."""
    from paper_2008_02734_b200.distributed import apportion, strip_ranges, _shard_idx
    assert apportion(8, [5, 5]) == [4, 4]
    assert sum(apportion(7, [9, 3, 1])) == 7 and min(apportion(7, [9, 3, 1])) >= 1
    for (M, N, kstop, H, parts) in [(1000, 900, 950, 128, 3), (5000, 300, 2650, 64, 4), (130, 140, 135, 128, 4)]:
        rng = strip_ranges(kstop, M, N, H, parts)
        rows = min(M, kstop + 1)
        S = (rows + H - 1) // H
        assert rng[0][0] == 0 and rng[-1][1] == S
        assert all(a <= b for a, b in rng) and all(rng[q][1] == rng[q + 1][0] for q in range(len(rng) - 1))
        # the shards' index ranges tile each of the last three diagonals exactly once
        for s3 in range(3):
            k = kstop - 2 + s3
            L_ = L.diag_length(k, M, N)
            seen = np.zeros(L_, int)
            for lo, hi in rng:
                a, b = _shard_idx(kstop, M, N, lo, hi, H)[s3]
                seen[a:b] += 1
            assert np.all(seen == 1)


def _batch_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2008_02734_b200.distributed import align_batch_distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pairs = [_pair(int(m), int(n), 3, 50 + t) for t, (m, n) in
                 enumerate(np.random.default_rng(4).integers(40, 400, size=(7, 2)))]
        done = []

        def oracle_batch(ps, cfg):  # test-only local compute: the C oracle per pair
            out = []
            for X, Y in ps:
                done.append((len(X), len(Y)))
                o = O.linmdtw(X.frames, Y.frames, min_dim=cfg.min_dim, precision=cfg.precision)
                out.append(L.AlignmentResult(
                    cost=o["cost"], path=o["path"], cells_processed=o["cells_processed"],
                    cells_budget=2 * len(X) * len(Y), precision="float32", algorithm="linmdtw",
                    peak_diag_values=o["peak_diag_values"], peak_table_cells=o["peak_table_cells"],
                    pivot_trace=o["pivot_trace"]))
            return out

        res = align_batch_distributed(pairs, min_dim=24, precision=32, aligner=oracle_batch)
        q.put((rank, [(r.cost, r.path, r.cells_processed, r.peak_diag_values, r.peak_table_cells,
                       list(r.pivot_trace)) for r in res], done))
    finally:
        dist.destroy_process_group()


def test_align_batch_distributed_gloo_world2():
    """BASELINE cfg4's multi-GPU sharding (pairs LPT-assigned to ranks, results
    exchanged as raw tensors): every rank returns every pair's result, equal
    to the single-process oracle, and each pair was aligned exactly once."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, res, done = q.get(timeout=300)
        got[rank] = (res, done)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pairs = [_pair(int(m), int(n), 3, 50 + t) for t, (m, n) in
             enumerate(np.random.default_rng(4).integers(40, 400, size=(7, 2)))]
    assert sorted(got[0][1] + got[1][1]) == sorted((len(X), len(Y)) for X, Y in pairs)
    for rank in (0, 1):
        for (X, Y), (cost, path, cells, pkd, pkt, trace) in zip(pairs, got[rank][0]):
            o = O.linmdtw(X, Y, min_dim=24, precision=32)
            assert cost == o["cost"] and np.array_equal(path, o["path"])
            assert cells == o["cells_processed"] and pkd == o["peak_diag_values"] and pkt == o["peak_table_cells"]
            assert trace == list(o["pivot_trace"])
