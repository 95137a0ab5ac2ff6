"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel.

usage: python tools/launch_summary.py launches.csv > profiles/rXX_launches_*.txt
"""
import csv, re, sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki])
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    tot[name] += v * scale
    cnt[name] += 1
all_us = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / cnt[k]:10.2f} {100 * tot[k] / all_us:6.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_us:12.1f}")
