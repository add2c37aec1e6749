"""Time the external path through ley_sort (one GPU) and through ley_sort_dist (NCCL, world size 1: the
multi-GPU external algorithm) on the same pinned host input. usage: dist_ext_time.py [n] [budget_bytes]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
budget = int(float(sys.argv[2])) if len(sys.argv) > 2 else (4 << 30) // 30
stage = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(stage.data_ptr(), n, 4, "uniform")
x = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
x.copy_(stage)
del stage
torch.cuda.empty_cache()
out = torch.empty_like(x).pin_memory()
out2 = torch.empty_like(x).pin_memory()
for rep in range(2):
    t0 = time.perf_counter(); ley.ley_sort(x, out, n, device_budget_bytes=budget); t1 = time.perf_counter()
    print(f"ley_sort external: {1e3 * (t1 - t0):.1f} ms", flush=True)
comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
for rep in range(2):
    t0 = time.perf_counter(); r = ley.ley_sort_dist(comm, x, n, out2, n, device_budget_bytes=budget); t1 = time.perf_counter()
    print(f"ley_sort_dist external (G=1): {1e3 * (t1 - t0):.1f} ms {r}", flush=True)
print("equal", torch.equal(out, out2))
ley.ley_comm_destroy(comm)
