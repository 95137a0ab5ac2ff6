"""Per-launch summary (time, DRAM bytes, L2 hit rate, occupancy, fp64 pipe, issue rate, launch
shape) from a raw-subset CSV written by tools/ncu_raw_subset.py.
usage: python tools/ncu_summary.py profiles/rXX_ncu_*_raw.csv > profiles/rXX_ncu_*_summary.csv"""
import csv
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread"]
rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
idx = [h.index(w) for w in WANT if w in h]
w = csv.writer(sys.stdout)
w.writerow([f"{h[i]} [{u[i]}]" if u[i] else h[i] for i in idx])
for r in rows[2:]:
    w.writerow([r[idx[0]].split("(")[0]] + [r[i] for i in idx[1:]])
