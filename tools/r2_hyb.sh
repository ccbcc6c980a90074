#!/bin/bash
# On the GPU box: hybrid fast/normal queues -- parity, per-level times, benches.
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/hyb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hyb_tests.log
for h in 1 0; do
  for cfg in cfg1 cfg2 cfg3; do
    echo "== $cfg hybrid=$h"
    LMDTW_HYBRID=$h timeout 300 python tools/probes/latency.py $cfg 2>&1 | python tools/probes/levels.py
  done
done > gpurun_out/hyb_levels.txt 2>&1
LMDTW_HOST_TIMING=1 python tools/probes/latency.py cfg3 2>&1 | grep sched | head -12 >> gpurun_out/hyb_levels.txt
LMDTW_HOST_TIMING=1 python tools/probes/latency.py cfg2 2>&1 | grep sched | head -8 >> gpurun_out/hyb_levels.txt
for c in cfg2 cfg3 cfg4 cfg5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 > gpurun_out/hy_$c.json; done
