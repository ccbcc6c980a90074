#!/bin/bash
# On the GPU box: cfg1 (fp64 d=2) per-item pace and pipelines-per-SM sweep.
for np in 0 1 2 4; do
  if [ $np = 0 ]; then unset LMDTW_ACTIVE_NP; else export LMDTW_ACTIVE_NP=$np; fi
  rm -f gpurun_out/tr_cfg1_$np.bin
  python tools/probes/trace_run.py cfg1 gpurun_out/tr_cfg1_$np.bin > /dev/null 2>&1
  echo "== cfg1 np=$np"
  python tools/probes/trace_strips.py gpurun_out/tr_cfg1_$np.bin 64 2>/dev/null | grep -E "^launch|run pace"
  timeout 120 python tools/probes/latency.py cfg1 2>&1 | python tools/probes/levels.py
done
