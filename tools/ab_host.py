"""A/B of library options on a host-memory sort (C5 scaled external path by default): ms per ley_sort.

usage: python tools/ab_host.py N BUDGET 'name:opt=v,...' ...
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1909_08006_b200 as ley

n = int(float(sys.argv[1]))
budget = int(float(sys.argv[2]))
x = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
out = torch.empty_like(x).pin_memory()
st = torch.empty(min(n, 50_000_000) * 100, dtype=torch.uint8, device="cuda")
for at in range(0, n, 50_000_000):
    m = min(50_000_000, n - at)
    gen.records_cuda(st.data_ptr(), m, 4, "uniform", i0=at)
    x[at * 100:(at + m) * 100].copy_(st[: m * 100])
del st
torch.cuda.empty_cache()
for v in sys.argv[3:]:
    name, _, spec = v.partition(":")
    opts = dict(kv.split("=") for kv in spec.split(",") if kv)
    old = {k: ley.ley_get_option(k) for k in opts}
    for k, val in opts.items():
        ley.ley_set_option(k, int(val))
    ley.ley_sort(x, out, n, device_budget_bytes=budget)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ley.ley_sort(x, out, n, device_budget_bytes=budget)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:12s} n={n} budget={budget} ms {[round(t, 1) for t in ts]} median {statistics.median(ts):.1f}", flush=True)
    for k, val in old.items():
        ley.ley_set_option(k, val)
