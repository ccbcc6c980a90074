#!/bin/bash
# On the GPU box: per-level times of cfg3 / cfg2 for tile-queue strip spacings.
for k in 32 64 128 256 512; do
  for cfg in cfg3 cfg2; do
    echo "== $cfg lag_key=$k"
    LMDTW_LAG_KEY=$k timeout 300 python tools/probes/latency.py $cfg 2>&1 | python tools/probes/levels.py
  done
done
