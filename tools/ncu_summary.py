"""Key metrics of every kernel in an ncu --set full report (speed-of-light, DRAM bytes, occupancy, issue,
top warp-stall reasons) as plain text for profiles/.

usage: python tools/ncu_summary.py report.ncu-rep [n_records]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
det = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h = det[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L2 Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Dynamic Shared Memory Per Block",
        "Block Size", "Grid Size"]
by = {}
for r in det[1:]:
    if len(r) <= h.index("Metric Value"):
        continue
    k = (r[h.index("ID")], r[h.index("Kernel Name")].split("(")[0])
    name = r[h.index("Metric Name")]
    if name in want:
        by.setdefault(k, {})[name] = f"{r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}".strip()
rh = raw[0]
rawby = {}
for r in raw[2:]:
    if len(r) < len(rh):
        continue
    rawby[r[rh.index("ID")]] = {rh[i]: r[i] for i in range(len(rh))}
for (i, k), m in by.items():
    print(f"== [{i}] {k}")
    for w in want:
        if w in m:
            print(f"   {w:36s} {m[w]}")
    rr = rawby.get(i, {})
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        def dram(key):
            return float(rr.get(key, "0").replace(",", "")) * scale.get(raw[1][rh.index(key)], 1.0)
        rd, wr = dram("dram__bytes_read.sum"), dram("dram__bytes_write.sum")
        if n:
            print(f"   DRAM bytes / record                  read {rd / n:.1f} + write {wr / n:.1f}")
    except (ValueError, IndexError):
        pass
    stalls = []
    for key, v in rr.items():
        if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print("   top stalls (warps per issue)        " + ", ".join(f"{s} {v:.2f}" for v, s in stalls[:6]))
