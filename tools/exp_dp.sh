#!/bin/bash
# On the GPU box: rebuild with each LMDTW_EXP value and measure probe 2 / 0 pace.
for e in "$@"; do
  LMDTW_NVCC_EXTRA="-DLMDTW_PROBES=1 -DLMDTW_EXP=$e" python paper_2008_02734_b200/build.py --force > /dev/null 2>&1 || { echo "build $e failed"; continue; }
  for m in 2 0; do
    echo "exp $e probe $m: $(LMDTW_PROBE=$m python tools/indep.py 32 12 | grep -E '=  592:')"
  done
done
