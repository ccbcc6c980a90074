#!/bin/bash
# On the GPU box: cfg1/cfg2/cfg3/cfg4 bench lines for latency-bound thresholds (LMDTW_LAT_FACTOR).
for f in 2.0 1.0 1.5 3.0 2.0; do
  for c in cfg2 cfg3 cfg1; do
    LMDTW_LAT_FACTOR=$f timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('factor $f', '$c', l['value'], l['ms_per_step'])"
  done
done
