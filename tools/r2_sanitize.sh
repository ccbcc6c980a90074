#!/bin/bash
# On the GPU box: compute-sanitizer memcheck / synccheck / racecheck of the
# small align and shard workloads (tools/probes/sanitize_case.py).
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for c in align shard; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/probes/sanitize_case.py $c \
      > gpurun_out/sanitize_${tool}_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_${c}.log
    echo "$tool $c: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' gpurun_out/sanitize_${tool}_${c}.log | tr '\n' ' ')"
  done
done
