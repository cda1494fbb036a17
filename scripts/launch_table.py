"""Per-launch table of an ncu launch-list CSV (gpu__time_duration, dram bytes): name, us, GB, B/pt."""
import csv
import sys

src = sys.argv[1]
npts = float(sys.argv[2]) if len(sys.argv) > 2 else 2560 * 1920 * 70
pat = sys.argv[3] if len(sys.argv) > 3 else ""
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[ii], {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
for k, d in sorted(per.items(), key=lambda kv: int(kv[0])):
    if pat and pat not in d["name"]:
        continue
    t = d["gpu__time_duration.sum"]
    rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
    print(f"{d['name'][:34]:34s} {t / 1e3:8.1f} us  read {rd / 1e9:6.2f} GB  write {wr / 1e9:5.2f} GB  "
          f"{(rd + wr) / npts:5.1f} B/pt  {(rd + wr) / t:6.0f} GB/s")
