"""Run `steps` ley_sort calls on a device-resident synthetic workload (for ncu / compute-sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import gen  # noqa: E402
import paper_1909_08006_b200 as ley  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e8)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--dist", default="uniform")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--l2", type=int, default=0)
ap.add_argument("--opt", action="append", default=[], help="library option NAME=VALUE (repeatable)")
a = ap.parse_args()
for kv in a.opt:
    k, v = kv.split("=")
    ley.ley_set_option(k, int(v))
n = int(a.n)
if a.l2:
    ley.ley_set_option("l2_fetch_bytes", a.l2)
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, a.seed, a.dist)
out = torch.empty_like(x)
for _ in range(a.warmup + a.steps):
    ley.ley_sort(x, out, n)
torch.cuda.synchronize()
print("ok", n)
