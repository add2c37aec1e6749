"""Time the G-rank distributed algorithm through the loopback transport on one GPU (all ranks' phases run
back to back; device copies stand in for NCCL). Per-rank work estimate = total / G."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 1, "uniform")
bounds = [r * n // G for r in range(G + 1)]
ins = [x[bounds[r] * 100: bounds[r + 1] * 100] for r in range(G)]
cap = n // G + 2
outs = [torch.empty(cap * 100, dtype=torch.uint8, device="cuda") for _ in range(G)]
args = (ins, [bounds[r + 1] - bounds[r] for r in range(G)], outs, [cap] * G)
for fused in (0, 1, 0, 1):
    ley.ley_set_option("dist_fused", fused)
    ley.ley_sort_dist_loopback(*args)
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        res = ley.ley_sort_dist_loopback(*args)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"dist_fused={fused} G={G} n={n}: best {best * 1e3:.2f} ms total, {best * 1e3 / G:.2f} ms per "
          f"rank-equivalent; n_out {[r[0] for r in res][:3]}...", flush=True)
ley.ley_set_option("dist_fused", 1)
