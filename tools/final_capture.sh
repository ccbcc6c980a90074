#!/bin/bash
# On the GPU box: the round's evidence -- GPU tests, default bench (with the
# CPU baseline), every BASELINE config, the reference arm, the launch list and
# one ncu --set full capture of the level-0 half-pass launch.
# Usage: tools/final_capture.sh TAG   (then here: python tools/write_profiles.py TAG rN)
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; tail -1 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-160
for c in cfg1 cfg2 cfg4 cfg5 cfg3x64 d100 d100x64; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  tail -1 gpurun_out/cfg_$c.json | cut -c1-160
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_reference.json 2>&1; tail -1 gpurun_out/final_reference.json | cut -c1-300
tools/profile.sh $TAG
