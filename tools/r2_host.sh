#!/bin/bash
# On the GPU box: full GPU suite, then phases and benches of the configs.
python -m pytest tests -m gpu -x -q > gpurun_out/host_tests.log 2>&1; echo "rc=$?" >> gpurun_out/host_tests.log
python tools/probes/latency.py cfg1 cfg2 cfg3 > gpurun_out/host_lat.txt 2>&1
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 > gpurun_out/h_$c.json; done
