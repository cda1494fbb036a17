"""Mean duration per kernel of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
d = collections.defaultdict(list)
for r in rows:
    name = re.sub(r"\(.*", "", r[ki]).replace("void eg::", "").replace("void ", "").strip()
    d[name].append(float(r[vi].replace(",", "")) * scale[r[ui]])
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:58]:58s} n={len(v):5d} mean={sum(v) / len(v):9.2f} us  share={100 * sum(v) / tot:5.1f} %")
