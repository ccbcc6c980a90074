#!/bin/bash
# On the GPU box: launch list of one bench step + one ncu --set full capture
# of the top (level-0) wave_kernel launch.  Usage: tools/profile.sh TAG [config]
TAG=${1:-prof}; CFG=${2:-cfg3}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu \
    > gpurun_out/launches_${TAG}.log 2>&1
LMDTW_WATCHDOG_S=300 ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 0 -c 1 \
    -o gpurun_out/${TAG} python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu \
    > gpurun_out/full_${TAG}.log 2>&1
tail -3 gpurun_out/full_${TAG}.log
