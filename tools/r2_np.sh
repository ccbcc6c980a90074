#!/bin/bash
for np in 3 2; do
  LMDTW_ACTIVE_NP=$np timeout 300 python tools/probes/latency.py cfg3 > gpurun_out/lat3_np$np.txt 2>&1
done
