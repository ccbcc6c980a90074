#!/bin/bash
# On the GPU box: rebuild with each "CH KC NP NS" tuple and measure the saturated pace.
while [ $# -ge 4 ]; do
  ch=$1; kc=$2; np=$3; ns=$4; shift 4
  LMDTW_NVCC_EXTRA="-DLMDTW_PROBES=1 -DLMDTW_CH=$ch -DLMDTW_KC=$kc -DLMDTW_NP=$np -DLMDTW_NS=$ns" python paper_2008_02734_b200/build.py --force > gpurun_out/build_$ch_$kc_$np.log 2>&1 || { echo "build $ch $kc $np failed"; tail -5 gpurun_out/build_$ch_$kc_$np.log; continue; }
  for m in 0 1 2; do
    echo "CH=$ch KC=$kc NP=$np NS=$ns probe $m: $(LMDTW_PROBE=$m python tools/probes/indep.py 32 12 | grep -E '=  592:')"
  done
done
