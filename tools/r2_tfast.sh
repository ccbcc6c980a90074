#!/bin/bash
for h in 0 1; do for cfg in cfg2 cfg3; do
  rm -f gpurun_out/tf_${cfg}_$h.bin
  LMDTW_HYBRID=$h python tools/probes/trace_run.py $cfg gpurun_out/tf_${cfg}_$h.bin > /dev/null 2>&1
  echo "== $cfg hybrid=$h"; python tools/probes/trace_fast.py gpurun_out/tf_${cfg}_$h.bin
done; done
