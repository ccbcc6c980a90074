#!/bin/bash
# On the GPU box: rebuild with each flag set and bench cfg5 (fp64 d=48).
for f in "$@"; do
  LMDTW_NVCC_EXTRA="$f" python paper_2008_02734_b200/build.py --force > gpurun_out/build_c5.log 2>&1 || { echo "build [$f] failed"; tail -3 gpurun_out/build_c5.log; continue; }
  timeout 600 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu > gpurun_out/c5.json 2>/dev/null
  echo "[$f] cfg5 $(tail -1 gpurun_out/c5.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"])')"
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
