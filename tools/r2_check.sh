#!/bin/bash
# On the GPU box: all GPU tests, then every config's bench (no CPU leg).
mkdir -p gpurun_out
T=${TAG:-c}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$T.log 2>&1; tail -1 gpurun_out/tests_$T.log
for c in cfg1 cfg2 cfg3 cfg3x64 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/${T}_$c.json 2>/dev/null
  echo "$c $(tail -1 gpurun_out/${T}_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
done
