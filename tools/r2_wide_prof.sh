#!/bin/bash
# On the GPU box: bench line of the default config (new roofline fields), and
# one ncu --set full capture of the level-0 WIDE wave_kernel at d = 100 fp32.
mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/wp_bench.log 2>&1; tail -1 gpurun_out/wp_bench.log | cut -c1-300
timeout 300 python bench.py --config d100 --steps 2 --warmup 1 --no-cpu > gpurun_out/wp_d100.log 2>&1; tail -1 gpurun_out/wp_d100.log | cut -c1-200
LMDTW_WATCHDOG_S=300 timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 0 -c 1 \
    -o gpurun_out/wide_d100 python bench.py --config d100 --steps 1 --warmup 0 --no-cpu > gpurun_out/wp_ncu.log 2>&1
tail -2 gpurun_out/wp_ncu.log
