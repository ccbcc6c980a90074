#!/bin/bash
# On the GPU box: probe builds with -D flag sets; independent-strip pace for probes 0/1/2.
for f in "$@"; do
  LMDTW_NVCC_EXTRA="-DLMDTW_PROBES=1 $f" python paper_2008_02734_b200/build.py --force > gpurun_out/build_exp.log 2>&1 || { echo "build [$f] failed"; tail -5 gpurun_out/build_exp.log; continue; }
  for m in 0 1 2; do
    echo "[$f] probe $m: $(LMDTW_PROBE=$m python tools/probes/indep.py 32 12 | grep -E 'strips=  592:')"
  done
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
