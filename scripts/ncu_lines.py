"""Aggregate ncu source-page stall samples per CUDA source line.
usage: python scripts/ncu_lines.py report.ncu-rep [kernel-regex] [topN]"""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg, tot = None, None, [], 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0].isdigit():
        i = hdr.index("Warp Stall Sampling (All Samples)")
        j = hdr.index("Instructions Executed")
        try:
            smp, ins = int(r[i]), int(r[j])
        except ValueError:
            continue
        tot += smp
        agg.append((smp, ins, f"{fname}:{r[0]}", r[1].strip()[:100]))
agg.sort(reverse=True)
print("total samples", tot)
for smp, ins, loc, src in agg[:top]:
    print(f"{smp:7d} {100.0 * smp / max(tot, 1):5.1f}% ins={ins:9d} {loc:22s} {src}")
