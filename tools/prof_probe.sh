#!/bin/bash
# On the GPU box: ncu --set full of the independent-strip run (probe build),
# for probe modes given as args (0 = full pipeline, 1 = cost warps alone, 2 = DP alone).
LMDTW_NVCC_EXTRA="-DLMDTW_PROBES=1 $EXTRA" python paper_2008_02734_b200/build.py --force > gpurun_out/build_probe.log 2>&1 || exit 1
for m in "$@"; do
  LMDTW_PROBE=$m LMDTW_WATCHDOG_S=300 ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 1 -c 1 \
    -o gpurun_out/probe${m}${TAG} python tools/probes/indep_one.py 32 12 592 20000 > gpurun_out/probe${m}${TAG}.log 2>&1
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
