"""Summarise an ncu report: SOL, occupancy, stall reasons, top SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(*a):
    return subprocess.run(["ncu", "-i", rep] + list(a), capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = rows[0]
keep = ("Duration", "SM Frequency", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Achieved Active Warps Per SM", "Registers Per Thread", "Grid Size", "Theoretical Occupancy",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "L1/TEX Hit Rate", "L2 Hit Rate",
        "DRAM Throughput", "Memory Throughput", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler")
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in keep:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
rh, rv = raw[0], raw[2]
st = []
for i, k in enumerate(rh):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((float(rv[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in st) or 1
print("stalls:", ", ".join(f"{k} {100 * v / tot:.1f}%" for v, k in sorted(st, reverse=True)[:10]))
for i, k in enumerate(rh):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed.sum", "smsp__inst_executed.sum", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
             "gpu__time_duration.sum"):
        print(f"{k:60s} {rv[i]} {raw[1][i]}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
sh = src[1]
ix = {k: i for i, k in enumerate(sh)}
data = src[2:]
col = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[ix[col]] or 0) for r in data) or 1
print(f"sass lines {len(data)}, samples {tot}")
for r in sorted(data, key=lambda r: -int(r[ix[col]] or 0))[:ntop]:
    print(f"{100 * int(r[ix[col]]) / tot:5.1f}% {r[ix['Source']][:100]}")
