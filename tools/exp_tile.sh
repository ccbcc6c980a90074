#!/bin/bash
# On the GPU box: rebuild with each tile width and bench cfg3 / cfg4 / cfg2.
for tw in "$@"; do
  LMDTW_NVCC_EXTRA="-DLMDTW_TILE_W=$tw" python paper_2008_02734_b200/build.py --force > gpurun_out/build_tile.log 2>&1 || { echo "build $tw failed"; continue; }
  for c in cfg3 cfg4 cfg2; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/tile${tw}_$c.json 2>/dev/null
    echo "TILE_W=$tw $c $(tail -1 gpurun_out/tile${tw}_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
  done
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
