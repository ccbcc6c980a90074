#!/bin/bash
# On the GPU box: sqrt exhaustive check, compute-sanitizer runs, full-size parity, bench.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sqrt_exhaustive tools/probes/sqrt_exhaustive.cu && \
  timeout 120 /tmp/sqrt_exhaustive > gpurun_out/sqrt_exhaustive.txt 2>&1
export LMDTW_WATCHDOG_S=600
for tool in memcheck racecheck synccheck; do
  for c in align shard; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/probes/sanitize_case.py $c \
      > gpurun_out/sanitize_${tool}_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_${c}.log
  done
done
unset LMDTW_WATCHDOG_S
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q --durations=20 > gpurun_out/fullsize.log 2>&1; echo rc=$? >> gpurun_out/fullsize.log
timeout 600 python bench.py > gpurun_out/bench_r2a.log 2>&1
