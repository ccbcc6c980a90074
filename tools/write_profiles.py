"""Summarise gpurun_out/ evidence of tools/final_capture.sh into profiles/<round>/final/.

    python tools/write_profiles.py [TAG] [ROUND]     (defaults: r1final r1)"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1final"
RND = sys.argv[2] if len(sys.argv) > 2 else "r1"
OUT = os.path.join(ROOT, "profiles", RND, "final")
G = os.path.join(ROOT, "gpurun_out")
os.makedirs(OUT, exist_ok=True)


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


# launch list of one bench step
rows = [r for r in csv.reader(open(os.path.join(G, f"launches_{TAG}.csv"))) if len(r) > 10 and r[0].isdigit()]
step = []
for r in rows:
    step.append((r[4].split("(")[0].replace("void ", ""), r[8], float(r[-1]) / 1e6))
    if "backtrace" in r[4]:
        break
tot = sum(t for _, _, t in step)
agg = {}
for n, _, t in step:
    agg[n] = agg.get(n, 0.0) + t
with open(os.path.join(OUT, "launch_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --config cfg3 --steps 1 "
            "--warmup 0 --no-cpu\nfirst alignment (one bench step, serialised launches, cold caches):\n")
    for n, g, t in step:
        f.write(f"  {t:9.3f} ms  grid {g:14s} {n}\n")
    f.write(f"  total {tot:.3f} ms\n")
    for n, t in sorted(agg.items(), key=lambda kv: -kv[1]):
        f.write(f"  share {100 * t / tot:5.1f}%  {n}\n")
subprocess.run(["cp", os.path.join(G, f"launches_{TAG}.csv"), os.path.join(OUT, "launches_cfg3.csv")])
rep = os.path.join(G, f"{TAG}.ncu-rep")
with open(os.path.join(OUT, "wave_kernel_level0_full.txt"), "w") as f:
    f.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "20"],
                           capture_output=True, text=True).stdout)
with open(os.path.join(OUT, "wave_kernel_level0_lines.txt"), "w") as f:
    f.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "30"],
                           capture_output=True, text=True).stdout)
# dram traffic of the level-0 launch
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, u, v = raw[0], raw[1], raw[2]


def metric(name):
    i = h.index(name)
    val = float(v[i].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[i], 1)
    return val * scale


rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
traffic = {"cfg3": {"launch": "wave_kernel<float,12,0> level 0 (1 node, fwd+rev half passes)",
                    "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "per_launch_bytes": int(rd + wr),
                    "cells": 10000299998, "algorithmic_bytes": 2 * 100000 * 12 * 4 + 6 * 100000 * 4,
                    "source": f"ncu --set full --clock-control none (profiles/{RND}/final/wave_kernel_level0_full.txt)"}}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "wave_kernel_traffic.json"), "w"), indent=1)
# every BASELINE config
res = []
for c, path in [("cfg1", "cfg_cfg1.json"), ("cfg2", "cfg_cfg2.json"), ("cfg3", "final_bench.json"),
                ("cfg4", "cfg_cfg4.json"), ("cfg5", "cfg_cfg5.json"), ("cfg3x64", "cfg_cfg3x64.json"),
                ("d100", "cfg_d100.json"), ("d100x64", "cfg_d100x64.json")]:
    if not os.path.exists(os.path.join(G, path)):
        continue
    d = last_json(os.path.join(G, path))
    res.append({"config": c, "workload": d["config"]["workload"], "dtype": d["dtype"], "GCUPS": d["value"],
                "ms_per_step": d["ms_per_step"], "sec_per_alignment": d["config"]["sec_per_alignment"],
                "e2e_GCUPS": d["e2e"]["value"], "wave_kernel_Gcell_s": d["roofline"]["achieved"],
                "roofline_frac_fp32_slots": d["roofline"]["frac"],
                "wave_kernel_computed_Gcell_s": d["roofline"].get("achieved_computed"),
                "frac_computed": d["roofline"].get("frac_computed"),
                "frac_alignment": d["roofline"].get("frac_alignment"), "clocks": d.get("clocks"),
                "cells_per_step": d["config"]["cells_per_step"],
                "cells_computed_per_step": d["config"].get("cells_computed_per_step")})
ref = last_json(os.path.join(G, "final_reference.json"))
json.dump({"gpu": "1x B200", "command": "python bench.py (cfg3) / --config <cfg> --steps 3 --warmup 1 --no-cpu",
           "results": res, "reference_arm": ref}, open(os.path.join(OUT, "configs.json"), "w"), indent=1)
for r in res:
    print(f"{r['config']:8s} {r['GCUPS']:9.3f} GCUPS  {r['ms_per_step']:9.3f} ms")
print("reference arm", ref["value"], ref["unit"], ref["cpu_baseline"]["cores"], "threads")
