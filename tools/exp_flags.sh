#!/bin/bash
# On the GPU box: for each quoted set of -D flags, rebuild (probe build) and
# measure the saturated pace for probes 0/1/2.
for f in "$@"; do
  LMDTW_NVCC_EXTRA="-DLMDTW_PROBES=1 $f" python paper_2008_02734_b200/build.py --force > gpurun_out/build_exp.log 2>&1 || { echo "build [$f] failed"; continue; }
  for m in 0 1 2; do
    echo "[$f] probe $m: $(LMDTW_PROBE=$m python tools/probes/indep.py 32 12 | grep -E '=  592:')"
  done
done
