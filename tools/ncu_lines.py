"""Warp-stall samples and executed instructions of one ncu report aggregated by CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
cur = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] != "":
        cur = (fname, r[0], r[1][:100])
        continue
    try:
        w, ins = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += w
    a[1] += ins
tw = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tw:5.1f}% stall {100 * v[1] / ti:5.1f}% inst  {k[0]}:{k[1]:>4}  {k[2]}")
