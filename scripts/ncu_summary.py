"""Summarise an ncu --set full report: per kernel duration, DRAM bytes / throughput, occupancy, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    print("=" * 100)
    print(name[:100])
    for k in KEYS:
        if k in h:
            print(f"  {k:60s} {r[h.index(k)]:>16s} {units[h.index(k)]}")
    st = [(h[i], float(r[i])) for i in range(len(h))
          if "average_warps_issue_stalled" in h[i] and h[i].endswith("per_issue_active.ratio") and r[i] not in ("", "n/a")]
    st.sort(key=lambda t: -t[1])
    print("  stalls/issue:", ", ".join(f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for n, v in st[:6]))
