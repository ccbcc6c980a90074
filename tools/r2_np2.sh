#!/bin/bash
# On the GPU box: per-level wave times of cfg2 / cfg3 with the active
# pipelines per SM forced (LMDTW_ACTIVE_NP) vs the default heuristic.
for cfg in cfg2 cfg3; do
  for np in 0 1 2 3 4; do
    if [ $np = 0 ]; then unset LMDTW_ACTIVE_NP; else export LMDTW_ACTIVE_NP=$np; fi
    echo "== $cfg np=$np"
    timeout 300 python tools/probes/latency.py $cfg 2>&1 | python tools/probes/levels.py
  done
done
