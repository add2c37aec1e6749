"""Per-stage DRAM traffic of one ley_sort call from ncu launch lists -> profiles/ncu_traffic.json.

usage: python tools/ncu_traffic.py CONFIG launches.csv n_records [CONFIG launches.csv n ...]
The csv comes from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`
over tools/profile_step.py (--warmup 1 --steps 1): the second call (from the second ka_tile_sort launch
on) is summarised. bench.py reads the file for roofline.traffic of the dominant stage.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = [("ka_tile", "K-a tile sort"), ("kb_", "K-b scan"), ("kc_plan_chunks", "K-b scan"),
         ("kc_", "K-c split"), ("kr_", "K-c' split"), ("kd_", "K-de sort+gather")]


def stage_of(name):
    for pre, st in STAGE:
        if pre in name:
            return st
    return None


def summarise(path, n):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = {h: i for i, h in enumerate(rows[start])}
    data = {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[hdr["ID"]]), r[hdr["Kernel Name"]])
        data.setdefault(key, {})[r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
    launches = sorted(data.items())
    firsts = [i for i, ((_, k), _) in enumerate(launches) if "ka_tile" in k]
    sel = launches[firsts[1]:] if len(firsts) > 1 else launches
    out = {}
    for (_, k), m in sel:
        st = stage_of(k)
        if st is None:
            continue
        e = out.setdefault(st, {"launches": 0, "bytes_per_launch": 0.0, "read": 0.0, "write": 0.0, "us": 0.0})
        e["launches"] += 1
        e["read"] += m.get("dram__bytes_read.sum", 0.0)
        e["write"] += m.get("dram__bytes_write.sum", 0.0)
        e["us"] += m.get("gpu__time_duration.sum", 0.0) / 1e3
    for st, e in out.items():
        e["bytes_per_launch"] = e["read"] + e["write"]  # all launches of the stage in one call
        e["bytes_per_record"] = round(e["bytes_per_launch"] / n, 2)
        e["read_per_record"] = round(e["read"] / n, 2)
        e["write_per_record"] = round(e["write"] / n, 2)
        e["us"] = round(e["us"], 1)
    return out


if __name__ == "__main__":
    dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    res = json.load(open(dst)) if os.path.exists(dst) else {}
    args = sys.argv[1:]
    for i in range(0, len(args), 3):
        cfg, path, n = args[i], args[i + 1], float(args[i + 2])
        res[cfg] = summarise(path, n)
        res[cfg]["_note"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one ley_sort call "
                             "(cold L2 per launch, serialised); bytes_per_launch sums the stage's launches")
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))
