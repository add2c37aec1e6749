"""Timeline of 6 consecutive ley_sort_submit calls of the C2 workload (LEY_TRACE_PIPE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LEY_TRACE_PIPE"] = "1"
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 1, "uniform")
hin = torch.empty(n * 100, dtype=torch.uint8).pin_memory(); hin.copy_(x); del x
hout = torch.empty_like(hin).pin_memory()
torch.cuda.empty_cache()
ley.ley_sort_submit(hin, hout, n); ley.ley_sort_drain()
for _ in range(6):
    ley.ley_sort_submit(hin, hout, n)
ley.ley_sort_drain()
