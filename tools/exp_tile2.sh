#!/bin/bash
for rep in 1 2; do
for tw in 2048 4096 8192; do
  LMDTW_NVCC_EXTRA="-DLMDTW_TILE_W=$tw" python paper_2008_02734_b200/build.py --force > gpurun_out/build_tile.log 2>&1 || { echo "build $tw failed"; continue; }
  for c in cfg3 cfg4; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu > gpurun_out/t2_${tw}_$c.json 2>/dev/null
    echo "rep $rep TILE_W=$tw $c $(tail -1 gpurun_out/t2_${tw}_$c.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"], l["roofline"]["frac"])')"
  done
done
done
python paper_2008_02734_b200/build.py --force > /dev/null 2>&1
