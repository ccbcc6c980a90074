#!/bin/bash
# On the GPU box: blocked-wait cycles by tag (LMDTW_WAITSTATS build) for cfg3 and cfg2.
LMDTW_NVCC_EXTRA="-DLMDTW_WAITSTATS=1" python paper_2008_02734_b200/build.py --force > gpurun_out/build_ws.log 2>&1 || exit 1
for c in cfg3 cfg2; do echo "== $c"; python tools/probes/waits_cfg.py $c; done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
