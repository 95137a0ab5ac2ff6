"""Compact raw-page CSV of an ncu report: every launch, the columns whose names start with one of
the prefixes below (time, DRAM/L2 traffic, occupancy, pipes, issue, stall reasons, launch shape).
usage: python tools/ncu_raw_subset.py report.ncu-rep > profiles/rXX_ncu_*_raw.csv"""
import csv, io, subprocess, sys

KEEP = ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct",
        "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "sm__warps_active.avg.pct", "sm__cycles_elapsed.max",
        "smsp__cycles_active.avg", "sm__inst_executed_pipe_fp64.avg.pct", "sm__inst_executed_pipe_lsu.avg.pct",
        "smsp__issue_active.avg.pct", "smsp__inst_executed.sum", "smsp__average_warps_issue_stalled",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit",
        "launch__waves_per_multiprocessor", "sm__maximum_warps_per_active_cycle_pct", "launch__cluster")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
cols = [i for i, name in enumerate(h) if any(name.startswith(k) for k in KEEP)]
w = csv.writer(sys.stdout)
for r in rows:
    w.writerow([r[i] if i < len(r) else "" for i in cols])
