#!/bin/bash
# On the GPU box: leaf-path parity, traces and timings.
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/leaf_tests.log 2>&1; echo "parity rc=$?" >> gpurun_out/leaf_tests.log
bash tools/probes/leaf_trace.sh > gpurun_out/leaf_trace2.txt 2>&1
python tools/probes/leaf_time.py > gpurun_out/leaf_time2.txt 2>&1
for c in cfg1 cfg2 cfg3; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 > gpurun_out/lf_$c.json; done
