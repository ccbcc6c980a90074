"""Stall reasons per code region (instructions grouped by execution count)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = rows[2:]
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data) or 1
g = defaultdict(lambda: defaultdict(int))
cnt = defaultdict(int)
for r in data:
    e = int(r[ix["Instructions Executed"]] or 0)
    cnt[e] += 1
    for k in reasons:
        g[e][k] += int(r[ix[k]] or 0)
    g[e]["all"] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
for e, d in sorted(g.items(), key=lambda x: -x[1]["all"])[:8]:
    top = sorted(((v, k) for k, v in d.items() if k != "all"), reverse=True)[:6]
    print(f"exec {e:>9d} x {cnt[e]:4d} instr: {100 * d['all'] / tot:5.1f}% of samples | "
          + ", ".join(f"{k[6:]} {100 * v / tot:.1f}" for v, k in top))
