import os, sys
sys.path.insert(0, "/root/repo"); os.environ["LEY_DEBUG_ALLOC"] = "1"
import torch, gen, paper_1909_08006_b200 as ley
n = 1_000_000; recs = gen.records(n, seed=44)
x = torch.from_numpy(recs).pin_memory(); out = torch.empty_like(x).pin_memory()
print(ley.ley_plan_query(n, 12 << 20), flush=True)
ley.ley_sort(x, out, n, device_budget_bytes=12 << 20)
print(ley.ley_device_bytes(), flush=True)
