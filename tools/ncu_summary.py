"""Summarise an ncu report: key SOL metrics + top SASS stall lines (used to write profiles/*.md)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = det[0]
want = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Avg. Active Threads Per Warp", "Achieved Occupancy",
        "Registers Per Thread", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Memory Throughput", "Branch Efficiency", "Theoretical Occupancy", "Grid Size", "Block Size"]
kname = None
for row in det[1:]:
    d = dict(zip(h, row))
    kname = d.get("Kernel Name", kname)
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:<40} {d['Metric Unit']:<12} {d['Metric Value']}")
print("kernel:", kname)
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
if raw:
    rh, units, vals = raw[0], raw[1], raw[2]
    for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
                "lts__t_requests_op_red.sum", "smsp__inst_executed_op_global_red.sum", "lts__t_sectors.sum",
                "gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]:
        for i, c in enumerate(rh):
            if c == key:
                print(f"{key:<55} {units[i]:<10} {vals[i]}")
    import re
    for i, c in enumerate(rh):   # pipe utilisation and reduction traffic
        if re.search(r"pipe_[a-z_]+(_cycles_active|inst_executed).*pct_of_peak_sustained_active$", c) or \
                re.search(r"^sm__inst_executed_pipe_[a-z_]+\.avg\.pct_of_peak_sustained_active$", c) or \
                re.search(r"op_red", c):
            try:
                if float(vals[i].replace(",", "")) > 1.0:
                    print(f"{c:<55} {units[i]:<10} {vals[i]}")
            except ValueError:
                pass
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
if len(src) > 2:
    sh = src[1]
    data = [dict(zip(sh, r)) for r in src[2:] if len(r) == len(sh)]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
    stall_cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    agg = {}
    for d in data:
        for c in stall_cols:
            agg[c] = agg.get(c, 0) + int(d[c] or 0)
    print("stall totals:", ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top]:
        st = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"{100*int(d['Warp Stall Sampling (All Samples)'])/tot:5.1f}% {d['Source'][:58]:<58} execd={d['Instructions Executed']:>10} thr={d['Avg. Threads Executed'][:4]} {st}")
