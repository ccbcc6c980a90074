#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_fullsize.py -k "wide or d100" -x -q > gpurun_out/tests_wide2.log 2>&1; tail -1 gpurun_out/tests_wide2.log
for c in d100 d100x64; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/w2_$c.json 2>/dev/null
  echo "$c $(tail -1 gpurun_out/w2_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
done
for w in 0 48 24; do
  LMDTW_WIDE_MIN=$w timeout 600 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu > gpurun_out/w2_cfg5_$w.json 2>/dev/null
  echo "cfg5 WIDE_MIN=$w $(tail -1 gpurun_out/w2_cfg5_$w.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"])')"
done
