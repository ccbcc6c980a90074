#!/bin/bash
# On the GPU box: rebuild with each poll backoff setting; bench cfg1 / cfg2 / cfg3 / cfg4.
for f in "$@"; do
  LMDTW_NVCC_EXTRA="$f" python paper_2008_02734_b200/build.py --force > gpurun_out/build_poll.log 2>&1 || { echo "build [$f] failed"; continue; }
  for c in cfg1 cfg2 cfg3 cfg4; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/poll.json 2>/dev/null
    echo "[$f] $c $(tail -1 gpurun_out/poll.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"])')"
  done
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
