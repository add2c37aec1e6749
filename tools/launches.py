"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel: us, B/record, GB/s."""
import csv
import sys

path = sys.argv[1]
n = float(sys.argv[2]) if len(sys.argv) > 2 else 1e8
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
data = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    key = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
    data.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
tot = 0.0
for (i, k), m in sorted(data.items()):
    t = m.get("gpu__time_duration.sum", 0.0)
    rd = m.get("dram__bytes_read.sum", 0.0)
    wr = m.get("dram__bytes_write.sum", 0.0)
    name = k.split("(")[0].replace("ley::<unnamed>::", "").replace("void ", "")[:40]
    if "gen_records" in k:
        continue
    tot += t
    print(f"{i:>3} {name:40s} {t / 1e3:9.1f} us  rd {rd / n:7.2f}  wr {wr / n:7.2f} B/rec  {(rd + wr) / t if t else 0:7.0f} GB/s")
print(f"sum {tot / 1e3:.1f} us")
