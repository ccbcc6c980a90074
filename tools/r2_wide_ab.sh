#!/bin/bash
# On the GPU box: for the default build and each quoted -D flag set, the WIDE
# (d > 64 fp32 / > 48 fp64) parity tests and d = 100 bench lines.
mkdir -p gpurun_out
for f in "" "$@"; do
  LMDTW_NVCC_EXTRA="$f" python paper_2008_02734_b200/build.py --force > gpurun_out/wab_build.log 2>&1 || { echo "build [$f] failed"; continue; }
  timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/wab_tests.log 2>&1; echo "[$f] $(tail -1 gpurun_out/wab_tests.log)"
  for c in d100 d100x64; do
    timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('[$f]', '$c', l['value'], l['ms_per_step'], l['roofline']['frac'])"
  done
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
