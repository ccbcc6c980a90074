#!/bin/bash
for sc in 0.25 0.5 0.75; do
  for cfg in cfg2 cfg3; do
    echo "== $cfg scale=$sc"
    LMDTW_FAST_SCALE=$sc timeout 300 python tools/probes/latency.py $cfg 2>&1 | python tools/probes/levels.py
  done
done
