"""Summarise an ncu launch-list CSV (gpu__time_duration, dram bytes) into per-kernel averages, the
share of the step, and profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py)."""
import csv
import json
import sys
from collections import defaultdict

src, out_txt, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per[r[ii]]["name"] = r[ki]
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    n = d["name"]
    if "eggen" in n:
        continue
    base = n.split("(")[0].replace("void ", "")
    a = agg[base]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
names = {"eg::k_update": "update_xr", "eg::k_stencil": None, "eg::k_thomas_tm": None, "eg::k_scale": "scale",
         "eg::k_start": "start", "eg::k_fin": "finalize"}
lines = [f"{'kernel':40s} {'launches':>8s} {'avg us':>10s} {'share':>7s} {'DRAM MB/launch':>15s} {'GB/s (ncu)':>11s}"]
traffic = {}
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    unit_t = t / n
    lines.append(f"{k:40s} {n:8d} {unit_t / 1e3:10.1f} {t / tot:7.3f} {b / n / 1e6:15.1f} {b / t:11.1f}")
    key = None
    if k.startswith("eg::k_update"):
        key = "update_xr"
    elif k.startswith("eg::k_stencil<1, 1>"):
        key = "stencil_dot_A"
    elif k.startswith("eg::k_stencil<1, 2>"):
        key = "stencil_dot_B"
    elif k.startswith("eg::k_thomas_tm<1, 1>"):
        key = "thomas_p"
    elif k.startswith("eg::k_thomas_tm<1, 2>"):
        key = "thomas_s"
    elif k.startswith("eg::k_scale"):
        key = "scale"
    elif k.startswith("eg::k_march<1, 1>"):
        key = "phase_A"
    elif k.startswith("eg::k_march<1, 2>"):
        key = "phase_B"
    if key:
        traffic[key] = b / n
open(out_txt, "w").write("\n".join(lines) + "\n")
json.dump({"mixed": traffic, "source": src}, open(out_json, "w"), indent=1)
print("\n".join(lines))
