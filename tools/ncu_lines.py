"""Top source lines of an ncu report by warp-stall samples (needs -lineinfo): tools/ncu_lines.py rep [n]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = next(x for x in r if x and x[0] == "Line No")
i = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
rows = [x for x in r if len(x) > i and x[0].isdigit() and x[i].isdigit()]
tot = sum(int(x[i] or 0) for x in rows) or 1
for x in sorted(rows, key=lambda x: -int(x[i] or 0))[:n]:
    print(f"{100 * int(x[i]) / tot:5.1f}% L{x[0]:>4} exec={x[ie]:>12} {x[1].strip()[:100]}")
