"""External path timeline (LEY_TRACE_EXT=1): C5-scaled workload, one warm + one traced call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
budget = int(sys.argv[2]) if len(sys.argv) > 2 else (4 << 30) // 3
x = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
st = torch.empty(50_000_000 * 100, dtype=torch.uint8, device="cuda")
for at in range(0, n, 50_000_000):
    m = min(50_000_000, n - at)
    gen.records_cuda(st.data_ptr(), m, 4, "uniform", i0=at)
    x[at * 100:(at + m) * 100].copy_(st[:m * 100])
del st; torch.cuda.empty_cache()
out = torch.empty_like(x).pin_memory()
ley.ley_sort(x, out, n, device_budget_bytes=budget)
os.environ["LEY_TRACE_EXT"] = "1"
print(ley.ley_plan_query(n, budget), flush=True)
t0 = time.perf_counter(); ley.ley_sort(x, out, n, device_budget_bytes=budget); print("wall", time.perf_counter() - t0)
