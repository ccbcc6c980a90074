#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2008_02734_b200/csrc -o /tmp/sqrt64 tools/probes/sqrt64_check.cu && timeout 300 /tmp/sqrt64 > gpurun_out/sqrt64_check.txt 2>&1; cat gpurun_out/sqrt64_check.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_f64.log 2>&1; tail -1 gpurun_out/tests_f64.log
for c in cfg1 cfg5 cfg3x64 d100x64 cfg3; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/f64_$c.json 2>/dev/null
  echo "$c $(tail -1 gpurun_out/f64_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
done
