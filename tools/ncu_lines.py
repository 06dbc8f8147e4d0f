"""Aggregate ncu warp-stall samples per CUDA source line (cuda,sass view).
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []
fname = ""
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or r[0] == "":
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    res.append((s, fname, r[0], r[1][:90]))
tot = sum(x[0] for x in res) or 1
for s, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:5s} {src}")
