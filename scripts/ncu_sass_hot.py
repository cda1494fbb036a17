"""Top SASS instructions of an ncu report by warp-stall samples (needs -lineinfo / --import-source).

    python scripts/ncu_sass_hot.py REPORT KERNEL_ID (e.g. ::regex:k_march:2) [N]
"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-id", kre], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
data, h = [], None
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        h = r
        continue
    if h and len(r) == len(h):
        try:
            float(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        data.append(r)
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
f = lambda r, i: float(r[i] or 0)
tot = sum(f(r, iss) for r in data)
print(f"samples {tot:.0f}, instructions {sum(f(r, iex) for r in data):.3e}")
for r in sorted(data, key=lambda r: -f(r, iss))[:n]:
    print(f"{r[0]:>6s} {100 * f(r, iss) / tot:5.1f}% {f(r, iex):12.0f}  {r[1][:100]}")
