#!/bin/bash
# On the GPU box: GPU tests, then benches under the latency-variant policies.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_lat.log 2>&1; tail -2 gpurun_out/tests_lat.log
for pol in 0 1 2; do
  for c in cfg1 cfg2 cfg3 cfg4; do
    LMDTW_LAT=$pol timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/lat${pol}_$c.json 2>/dev/null
    echo "LAT=$pol $c $(tail -1 gpurun_out/lat${pol}_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
  done
done
for c in cfg1 cfg2 cfg3; do
  LMDTW_LAT_LEAF=1 timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/latleaf_$c.json 2>/dev/null
  echo "LAT_LEAF=1 $c $(tail -1 gpurun_out/latleaf_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
done
