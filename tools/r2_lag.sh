#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -x -q > gpurun_out/tests_lag.log 2>&1; tail -1 gpurun_out/tests_lag.log
for k in 128 64 256; do
  for c in cfg3 cfg2 cfg4; do
    LMDTW_LAG_KEY=$k timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/lag${k}_$c.json 2>/dev/null
    echo "LAG_KEY=$k $c $(tail -1 gpurun_out/lag${k}_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
  done
done
