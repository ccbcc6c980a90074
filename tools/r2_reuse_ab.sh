#!/bin/bash
for ru in 0 1; do
  for c in cfg2 cfg3 cfg4; do
    LMDTW_REUSE=$ru timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/ab.json 2>/dev/null
    echo "REUSE=$ru $c $(tail -1 gpurun_out/ab.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"], l["roofline"]["achieved"], l["config"]["cells_computed_per_step"])')"
  done
done
for ru in 0 1; do LMDTW_REUSE=$ru timeout 300 python tools/probes/latency.py cfg2 > gpurun_out/lat_ru$ru.txt 2>&1; done
