#!/bin/bash
# On the GPU box: WIDE (d > 64 fp32 / > 48 fp64) parity tests and d = 100
# bench lines for the default build, then for each quoted -D flag set.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/wab_tests.log 2>&1; tail -2 gpurun_out/wab_tests.log
for c in d100 d100x64; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('default', '$c', l['value'], l['ms_per_step'], l['roofline']['frac'])"
done
for f in "$@"; do
  LMDTW_NVCC_EXTRA="$f" python paper_2008_02734_b200/build.py --force > gpurun_out/wab_build.log 2>&1 || { echo "build [$f] failed"; continue; }
  for c in d100 d100x64; do
    timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('[$f]', '$c', l['value'], l['ms_per_step'], l['roofline']['frac'])"
  done
done
