"""Stall-reason totals over the SASS instructions of one kernel whose execution count lies in a
range (e.g. the body of a hot loop), from an ncu --set full report with source counters.

    python scripts/ncu_stalls_range.py REPORT KERNEL_ID LO HI
"""
import csv
import subprocess
import sys
from collections import Counter

rep, kid, lo, hi = sys.argv[1], sys.argv[2], float(sys.argv[3]), float(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-id", kid],
                     capture_output=True, text=True).stdout
h, tot, ops, n = None, Counter(), Counter(), 0
for r in csv.reader(out.splitlines()):
    if len(r) > 3 and r[0] == "Address":
        h = r
        continue
    if not h or len(r) != len(h):
        continue
    try:
        ex = float(r[h.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    if not (lo <= ex <= hi):
        continue
    n += 1
    op = r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]
    ops[op.split(".")[0]] += 1
    for i, c in enumerate(h):
        if c.startswith("stall_") and "Not Issued" not in c:
            tot[c] += float(r[i] or 0)
s = sum(tot.values()) or 1
print(f"{n} instructions in range; samples {s:.0f}")
for k, v in tot.most_common(12):
    print(f"  {k:26s} {100 * v / s:5.1f}%")
print("opcodes:", ", ".join(f"{k}:{v}" for k, v in ops.most_common(25)))
