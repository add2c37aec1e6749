"""Average per-stage times of ley_sort on a device-resident synthetic workload (A/B of library variants
via LEY_LIBRARY_OVERRIDE)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
dist = sys.argv[2] if len(sys.argv) > 2 else "uniform"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 1, dist)
out = torch.empty_like(x)
for _ in range(2):
    ley.ley_sort(x, out, n)
ley.ley_set_option("profile", 1)
acc = {}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    ley.ley_sort(x, out, n)
    for k, v in ley.ley_stage_times()[0]:
        acc.setdefault(k, []).append(v)
e1.record(); torch.cuda.synchronize()
tag = os.path.basename(os.environ.get("LEY_LIBRARY_OVERRIDE", "default"))
print(tag, f"total {e0.elapsed_time(e1)/steps:.3f} ms", {k: round(statistics.mean(v), 3) for k, v in acc.items()})
