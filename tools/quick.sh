#!/bin/bash
# On the GPU box: GPU tests, one bench run, launch list of one bench step.  Usage: tools/quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/tests_${TAG}.log 2>&1; tail -3 gpurun_out/tests_${TAG}.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}.log 2>&1; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-400
LMDTW_WATCHDOG_S=100 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")) if len(r) > 10 and r[0].isdigit()]
print(" ".join(f"{float(r[-1])/1e6:.3f}" for r in rows if "wave" in r[4])[:400])
PY
