#!/bin/bash
# On the GPU box: cfg5 / d=100 throughput, WIDE switch-over experiments.
mkdir -p gpurun_out
for w in 0 48 24; do
  LMDTW_WIDE_MIN=$w timeout 600 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu > gpurun_out/wide${w}_cfg5.json 2>/dev/null
  echo "WIDE_MIN=$w cfg5 $(tail -1 gpurun_out/wide${w}_cfg5.json | cut -c1-220)"
done
for c in d100 d100x64 cfg3x64; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/b_$c.json 2>/dev/null
  echo "$c $(tail -1 gpurun_out/b_$c.json | cut -c1-220)"
done
