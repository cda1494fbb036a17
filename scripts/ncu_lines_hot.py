"""Warp-stall samples and executed instructions of one kernel aggregated per CUDA source line.

    python scripts/ncu_lines_hot.py REPORT KERNEL_ID [N]      (KERNEL_ID e.g. ::regex:k_march:2)
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kid = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-id", kid], capture_output=True, text=True).stdout
h, fname = None, "?"
agg = defaultdict(lambda: [0.0, 0.0, ""])
reasons = defaultdict(float)
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        h = r
        continue
    if not h or len(r) != len(h):
        continue
    try:
        s = float(r[4] or 0)
        ex = float(r[h.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    a = agg[(fname, int(r[0]) if r[0].isdigit() else 0)]
    a[0] += s
    a[1] += ex
    a[2] = r[1]
tot = sum(v[0] for v in agg.values()) or 1.0
print(f"samples {tot:.0f}  instructions {sum(v[1] for v in agg.values()):.3e}")
for (f, ln), (s, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{f:14s}{ln:5d} {100 * s / tot:5.1f}% {ex:13.0f}  {src.strip()[:90]}")
