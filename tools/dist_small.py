"""Per-phase times of the NCCL dist path at world size 1 with the exchange phases forced on, for a per-rank
slice of C2 at G ranks (n = 1e8 / G): the fixed costs a rank pays at 8 GPUs. usage: dist_small.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 12_500_000
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 1, "uniform")
out = torch.empty_like(x)
comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
for g1 in (0, 1):
    ley.ley_set_option("dist_exchange_g1", g1)
    for _ in range(3):
        ley.ley_sort_dist(comm, x, n, out, n)
    torch.cuda.synchronize()
    ley.ley_set_option("profile", 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ley.ley_sort_dist(comm, x, n, out, n)
    e1.record()
    torch.cuda.synchronize()
    st, nl = ley.ley_stage_times()
    ley.ley_set_option("profile", 0)
    print(f"exchange_g1={g1} n={n}: {e0.elapsed_time(e1) / 10:.3f} ms/call; last call stages "
          f"{[(a, round(b, 3)) for a, b in st]}; launches {nl}", flush=True)
ley.ley_comm_destroy(comm)
