"""Per-level durations from LMDTW_PHASES output (stdin): launched -> done."""
import re
import sys
t_launch = None
out = []
for line in sys.stdin:
    if "ms per alignment" in line:
        print(line.strip())
    m = re.match(r"lmdtw phase (.+?)\s+([\d.]+) us", line.strip())
    if not m:
        continue
    what, t = m.group(1).strip(), float(m.group(2))
    if what == "batch launched":
        t_launch = t
    elif what == "batch done" and t_launch is not None:
        out.append(t - t_launch)
    elif what == "leaves done":
        out.append(-(t - prev))
    prev = t
print("  levels (ms):", " ".join(f"{x / 1e3:.3f}" for x in out))
