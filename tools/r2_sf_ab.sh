#!/bin/bash
# On the GPU box: full GPU tests, cfg1/cfg2/cfg3 bench lines, ncu of the d=100
# WIDE level-0 launch (default build), then the same benches with each quoted
# -D flag set.
mkdir -p gpurun_out
b() { timeout 300 python bench.py --config $1 --steps ${2:-3} --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$3', '$1', l['value'], l['ms_per_step'], l['roofline']['frac'])"; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/sf_tests.log 2>&1; tail -2 gpurun_out/sf_tests.log
for c in cfg3 cfg2 cfg1; do b $c 5 default; done
LMDTW_WATCHDOG_S=300 timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 0 -c 1 \
    -o gpurun_out/wide2_d100 python bench.py --config d100 --steps 1 --warmup 0 --no-cpu > gpurun_out/sf_ncu.log 2>&1
for f in "$@"; do
  LMDTW_NVCC_EXTRA="$f" python paper_2008_02734_b200/build.py --force > gpurun_out/sf_build.log 2>&1 || { echo "build [$f] failed"; continue; }
  for c in cfg3 cfg2 cfg1; do b $c 5 "[$f]"; done
done
