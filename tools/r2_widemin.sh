#!/bin/bash
# On the GPU box: bench lines with the WIDE kernels taking over at lower d (LMDTW_WIDE_MIN).
mkdir -p gpurun_out
b() { timeout 400 env $3 python bench.py --config $1 --steps ${2} --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys
try:
    l=json.loads(sys.stdin.read()); print('[$3]', '$1', l['value'], l['ms_per_step'], l['roofline']['frac'])
except Exception: print('[$3] $1 failed')"; }
for e in "X=0" "LMDTW_WIDE_MIN=40" "LMDTW_WIDE_MIN=20"; do b cfg5 3 $e; done
for e in "X=0" "LMDTW_WIDE_MIN=12"; do b cfg3x64 3 $e; b cfg3 3 $e; done
