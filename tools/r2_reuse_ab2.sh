#!/bin/bash
for env in "LMDTW_REUSE=0" "LMDTW_WINDOWS=2" "LMDTW_WINDOWS=1"; do
  for c in cfg2 cfg3 cfg4 cfg5; do
    env $env timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/ab.json 2>/dev/null
    echo "$env $c $(tail -1 gpurun_out/ab.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"], l["config"]["cells_computed_per_step"])')"
  done
done
