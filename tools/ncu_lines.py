"""Summarise an ncu report's source page: top CUDA source lines by warp-state samples.

usage: python tools/ncu_lines.py report.ncu-rep [N] [launch index]
"""
import csv, io, os, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
extra = ["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + extra,
                     capture_output=True, text=True).stdout
data, fname, hdr = [], "", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        ins = r[hdr.index("Instructions Executed")]
    except (ValueError, IndexError):
        continue
    data.append((samp, f"{fname}:{r[0]}", ins, r[1].strip()[:95]))
tot = sum(d[0] for d in data) or 1
print("total samples", int(tot))
for s, loc, ins, src in sorted(data, reverse=True)[:top]:
    print(f"{int(s):7d} {100 * s / tot:5.1f}% {loc:>22} ins={ins:>9} {src}")
