"""Hottest CUDA source lines of one kernel in an ncu report, by warp-stall samples.

usage: python tools/ncu_hot.py report.ncu-rep <kernel-regex> [top]
(needs the binary compiled with -lineinfo and the report captured with --import-source on)
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}", "-s", skip, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = "?"
data = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    if len(r) > 4 and r[2] == "-":
        try:
            s = int(r[4])
        except ValueError:
            continue
        data.append((s, f"{cur_file}:{r[0]}", r[1].strip()[:100]))
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}")
for s, l, t in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {l:>22}  {t}")
