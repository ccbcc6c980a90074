#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/bt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bt_tests.log
python tools/probes/latency.py cfg1 cfg2 cfg3 2>&1 | grep "ms per" > gpurun_out/bt_lat.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/bt_cfg1.csv python bench.py --config cfg1 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
