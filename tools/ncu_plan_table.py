"""Per-launch table of an ncu report (config-2 plan kernels): DRAM bytes, time, grid,
registers, occupancy, instructions, issue activity.  usage: ncu_plan_table.py REP TITLE"""
import csv
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
M = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__grid_size",
     "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
print(f"# ncu --set full --clock-control none: {title}")
print("kernel | " + " | ".join(f"{m} [{u[h.index(m)]}]" for m in M))
for r in rows[2:]:
    k = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    print(k + " | " + " | ".join(r[h.index(m)] for m in M))
