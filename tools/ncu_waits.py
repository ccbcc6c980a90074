"""Stall samples on every mbarrier try-wait / branch-back instruction, keyed by the
barrier's shared-memory offset (which ring/queue it is)."""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}
data = rows[2:]
col = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[ix[col]] or 0) for r in data) or 1
agg = {}
last_bar = None
for r in data:
    src = r[ix["Source"]]
    m = re.search(r"TRYWAIT.*\[(R\d+)\+URZ\+(0x[0-9a-f]+)\]", src)
    if m:
        last_bar = m.group(2)
    n = int(r[ix[col]] or 0)
    if last_bar and ("TRYWAIT" in src or "BRA" in src):
        agg[last_bar] = agg.get(last_bar, 0) + n
    if "BRA" in src and "TRYWAIT" not in src:
        pass
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"barrier smem +{k}: {100 * v / tot:5.1f}% of samples")
