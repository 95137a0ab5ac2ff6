"""Print selected raw metrics per launch from an ncu report as a clean CSV.

usage: python tools/ncu_metrics.py report.ncu-rep metric1,metric2,...
"""
import csv, io, re, subprocess, sys

rep, mets = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", mets], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
want = mets.split(",")
w = csv.writer(sys.stdout)
w.writerow(["kernel"] + [f"{m} [{u[h.index(m)]}]" for m in want if m in h])
for r in rows[2:]:
    w.writerow([re.sub(r"\(.*", "", r[h.index("Kernel Name")])] + [r[h.index(m)] for m in want if m in h])
