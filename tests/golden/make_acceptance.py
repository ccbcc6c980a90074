"""Golden vectors for the reference's acceptance criterion 1 (exactness sweep),
generated from the REAL reference.  Run here (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_acceptance.py

The sweep is /root/reference/pkg/tests/test_acceptance.py:40-74: dims {1, 4},
M, N in 2..12, 9 repetitions -> 2,178 instances, X = random_series(M, dim,
seed), Y = random_series(N, dim, seed + 7), linmdtw(min_dim=2).  The reference
certifies each result with OptimalPathDag (brute-force optimal-cell DAG); this
script stores, per instance, that certified minimum cost and the reference's
own linmdtw result (cost, path, pivot trace) in fp64 and fp32, so the GPU box
can replay the sweep without the reference.  Inputs are regenerated from the
seeds (numpy default_rng standard_normal, cast to float32 by FeatureSeries).
"""
from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import lmdtw  # noqa: E402  (the reference package)
from lmdtw import OptimalPathDag  # noqa: E402
from lmdtw.synth import random_series  # noqa: E402

KEYS = ("i", "j", "i_off", "j_off", "M", "N", "sub_i", "sub_j", "diagonal_k")


def instances():
    for dim in (1, 4):
        for M in range(2, 13):
            for N in range(2, 13):
                for rep in range(9):
                    yield dim, M, N, rep, 1_000_000 * dim + 10_000 * M + 100 * N + rep


def main():
    meta, dag_cost = [], []
    cost = {32: [], 64: []}
    paths = {32: [], 64: []}
    plen = {32: [], 64: []}
    piv = {32: [], 64: []}
    ptot = {32: [], 64: []}
    npiv = {32: [], 64: []}
    for dim, M, N, rep, seed in instances():
        X = random_series(M, dim, seed)
        Y = random_series(N, dim, seed + 7)
        meta.append((dim, M, N, rep, seed))
        dag_cost.append(OptimalPathDag(X, Y).min_cost)
        for prec in (32, 64):
            r = lmdtw.linmdtw(X, Y, min_dim=2, precision=prec)
            cost[prec].append(r.cost)
            paths[prec].append(np.asarray(r.path, np.int16))
            plen[prec].append(len(r.path))
            npiv[prec].append(len(r.pivot_trace))
            for e in r.pivot_trace:
                piv[prec].append([int(e[k]) for k in KEYS])
                ptot[prec].append(float(e["total_at_pivot"]))
    out = {"meta": np.asarray(meta, np.int64), "dag_cost": np.asarray(dag_cost, np.float64)}
    for prec in (32, 64):
        out[f"cost{prec}"] = np.asarray(cost[prec], np.float64)
        out[f"path{prec}"] = np.concatenate(paths[prec])
        out[f"plen{prec}"] = np.asarray(plen[prec], np.int32)
        out[f"piv{prec}"] = np.asarray(piv[prec], np.int32).reshape(-1, len(KEYS))
        out[f"ptot{prec}"] = np.asarray(ptot[prec], np.float64)
        out[f"npiv{prec}"] = np.asarray(npiv[prec], np.int32)
    np.savez_compressed(os.path.join(HERE, "acceptance_c1.npz"), **out)
    print(f"{len(meta)} instances; fp64 cost == certified minimum: "
          f"{int(np.sum(out['cost64'] == out['dag_cost']))}")


if __name__ == "__main__":
    main()
