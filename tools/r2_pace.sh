#!/bin/bash
# On the GPU box: per-item DP pace of cfg2's and cfg3's first launches with 1, 2, 4 pipelines per SM.
for np in 1 2 4; do
  for cfg in cfg2 cfg3; do
    rm -f gpurun_out/tr_${cfg}_$np.bin
    LMDTW_ACTIVE_NP=$np python tools/probes/trace_run.py $cfg gpurun_out/tr_${cfg}_$np.bin > /dev/null 2>&1
    echo "== $cfg np=$np"
    python tools/probes/trace_strips.py gpurun_out/tr_${cfg}_$np.bin 2>/dev/null | grep -E "^launch [0-3] |run pace" | head -8
  done
done
