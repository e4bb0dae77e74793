"""Summary of an ncu report: per launch duration, DRAM bytes, throughputs,
issue activity, instructions and the top warp-stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:60]
    d = {k.split("__")[1][:28]: f"{r[h.index(k)]} {units[h.index(k)]}".strip() for k in keys if k in h}
    print(name, d)
    st = sorted(((h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i] or 0))
                 for i in range(len(h)) if "pcsamp_warps_issue_stalled" in h[i]
                 and not h[i].endswith("not_issued")), key=lambda x: -x[1])
    print("   stalls:", ", ".join(f"{k} {int(v)}" for k, v in st[:8]))
