"""Summarise an ncu --set full report: one row per profiled launch with the
metrics the round notes cite.  python profiles/scripts/ncu_summary.py rep.ncu-rep > out.csv"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "smsp__inst_executed.sum"]

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = csv.writer(sys.stdout)
out.writerow(["kernel"] + [f"{k} [{units[hdr.index(k)]}]" if k in hdr else k for k in KEYS])
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "").split("(")[0].replace("void ", "")
    out.writerow([name] + [d.get(k, "") for k in KEYS])
