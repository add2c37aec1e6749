"""Per-kernel DRAM table from the committed ncu launch lists (SURVEY §8d "ncu evidence"): for the second
ley_sort call of each config, every kernel's summed duration, DRAM bytes, bytes per record, achieved GB/s
and its fraction of the measured copy peak (MEASURED_PEAKS.json) and of the 8 TB/s nominal HBM3e peak.
usage: python tools/kernel_table.py [round] > profiles/rNN_kernel_table.md"""
import csv
import json
import os
import re
import sys

ROUND = sys.argv[1] if len(sys.argv) > 1 else "r02"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = {"c1": 1e6, "c2": 1e8, "c3": 2e8, "c4": 6e8}
peak = 6456.8
p = os.path.join(ROOT, "MEASURED_PEAKS.json")
if os.path.exists(p):
    peak = float(json.load(open(p)).get("hbm_gbs", peak))


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name)
    return re.sub(r"ley::(<unnamed>|\(anonymous namespace\))::", "", name)


print(f"# Per-kernel DRAM traffic and rate (ncu, 2nd ley_sort call; peak {peak} GB/s measured, 8000 nominal)\n")
for c, n in CFG.items():
    f = os.path.join(ROOT, "profiles", f"{ROUND}_launches_{c}.csv")
    if not os.path.exists(f):
        continue
    rows = list(csv.reader(open(f)))
    st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = {k: i for i, k in enumerate(rows[st])}
    per = {}
    order = []
    for r in rows[st + 1:]:
        key = (r[h["ID"]], r[h["Kernel Name"]])
        if key not in per:
            per[key] = {}
            order.append(key)
        per[key][r[h["Metric Name"]]] = (float(r[h["Metric Value"]].replace(",", "")), r[h["Metric Unit"]])
    ka = [i for i, k in enumerate(order) if "ka_tile" in k[1]]
    order = order[ka[1]:] if len(ka) > 1 else order
    agg = {}
    for k in order:
        m = per[k]
        t = m.get("gpu__time_duration.sum", (0, "ns"))
        tns = t[0] * (1e3 if t[1] == "us" else 1e6 if t[1] == "ms" else 1)
        def b(name):
            v, u = m.get(name, (0, "byte"))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        name = short(k[1])
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += tns
        a[2] += b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
    print(f"## {c.upper()} (n = {n:.0e})\n")
    print("| kernel | launches | time (us) | DRAM bytes/record | GB/s | of measured peak | of 8 TB/s |")
    print("|---|---|---|---|---|---|---|")
    tot_t = tot_b = 0
    for name, (cnt, tns, byt) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        tot_t += tns
        tot_b += byt
        gbs = byt / tns if tns else 0
        print(f"| `{name}` | {cnt} | {tns / 1e3:.1f} | {byt / n:.1f} | {gbs:.0f} | {gbs / peak:.2f} | {gbs / 8000:.2f} |")
    gbs = tot_b / tot_t
    print(f"| **all** | | {tot_t / 1e3:.1f} | {tot_b / n:.1f} | {gbs:.0f} | {gbs / peak:.2f} | {gbs / 8000:.2f} |\n")
