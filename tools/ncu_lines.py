"""Stall samples aggregated per CUDA source line (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[2]
ix = {}
for i, k in enumerate(h):
    ix.setdefault(k, i)
col = "Warp Stall Sampling (All Samples)"
lines = []
for r in rows[3:]:
    if len(r) > ix[col] and r[0] and r[ix[col]] not in ("", "-"):
        try:  # multi-line inline asm breaks ncu's CSV quoting: skip those rows
            lines.append((int(r[ix[col]]), int(r[ix["Instructions Executed"]] or 0), r[0], r[1].strip()))
        except ValueError:
            pass
tot = sum(v[0] for v in lines) or 1
for s, e, ln, src in sorted(lines, reverse=True)[:ntop]:
    print(f"{100 * s / tot:5.1f}% L{ln:>5} exec={e:>12} {src[:90]}")
