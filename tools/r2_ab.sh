#!/bin/bash
# On the GPU box: A/B of build flags.  Usage: tools/r2_ab.sh "CONFIGS" "FLAGS1" "FLAGS2" ...
# ("" = the default build; every flag set gets the GPU tests of TESTS, if set).
mkdir -p gpurun_out
CFGS=$1; shift
for f in "$@"; do
  LMDTW_NVCC_EXTRA="$f" python paper_2008_02734_b200/build.py --force > gpurun_out/ab_build.log 2>&1 || { echo "build [$f] failed"; continue; }
  if [ -n "$TESTS" ]; then timeout 1200 python -m pytest $TESTS -x -q > gpurun_out/ab_tests.log 2>&1; echo "[$f] $(tail -1 gpurun_out/ab_tests.log)"; fi
  for c in $CFGS; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu > gpurun_out/ab_line.log 2>&1
    tail -1 gpurun_out/ab_line.log | python -c "import json,sys
try:
    l=json.loads(sys.stdin.read()); print('[$f]', '$c', l['value'], l['ms_per_step'], l['roofline']['frac'])
except Exception as e: print('[$f] $c failed')"
  done
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
