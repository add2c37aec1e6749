"""One NCCL communicator of one rank running the full dist path (splitters, K-p, exchange, local sort) on
n uniform records: for ncu captures of the dist kernels (K-s0, K-p). usage: dist_step.py [n] [fused] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
fused = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ley.ley_set_option("dist_exchange_g1", 1)
ley.ley_set_option("dist_fused", fused)
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 1, "uniform")
out = torch.empty_like(x)
comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
for _ in range(reps):
    ley.ley_sort_dist(comm, x, n, out, n)
torch.cuda.synchronize()
ley.ley_comm_destroy(comm)
print("ok")
