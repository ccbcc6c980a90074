#!/bin/bash
# On the GPU box: per-item traces of cfg3's launches (leaves last) and of one
# 2000x2000 dtw_full, analysed by trace_strips.py.
rm -f gpurun_out/trace_cfg3.bin gpurun_out/trace_full.bin
python tools/probes/trace_run.py cfg3 gpurun_out/trace_cfg3.bin > /dev/null
python tools/probes/trace_strips.py gpurun_out/trace_cfg3.bin | tail -12
python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import bench, paper_2008_02734_b200 as L
for (M, prec, d) in [(2000, 32, 12), (500, 64, 2)]:
    X, Y = bench.latent_pair(M, M, d, seed=1)
    L.dtw_full(X, Y, precision=prec)
    os.environ["LMDTW_TRACE_FILE"] = f"gpurun_out/trace_full{M}.bin"
    L.dtw_full(X, Y, precision=prec)
    os.environ.pop("LMDTW_TRACE_FILE")
PY
python tools/probes/trace_strips.py gpurun_out/trace_full2000.bin
python tools/probes/trace_strips.py gpurun_out/trace_full500.bin 64
