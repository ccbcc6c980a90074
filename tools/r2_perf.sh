#!/bin/bash
# On the GPU box: GPU tests, default bench, per-config benches, latency breakdown.
mkdir -p gpurun_out
T=${TAG:-p}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$T.log 2>&1; tail -2 gpurun_out/tests_$T.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -1 gpurun_out/bench_$T.json | cut -c1-300
for c in cfg1 cfg2 cfg4 cfg5 cfg3x64; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/cfg_${c}_$T.json 2> gpurun_out/cfg_${c}_$T.err
  tail -1 gpurun_out/cfg_${c}_$T.json | cut -c1-200
done
timeout 300 python tools/probes/latency.py cfg1 cfg2 > gpurun_out/latency_$T.txt 2>&1
