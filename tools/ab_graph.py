"""Alternate graphs on/off at one size (plain timing, no stage events): are graph replays slower anywhere?"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1909_08006_b200 as ley

n = int(float(sys.argv[1]))
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 3, "uniform")
out = torch.empty_like(x)
res = {0: [], 1: []}
for g in (1, 0):
    ley.ley_set_option("graphs", g)
    ley.ley_sort(x, out, n)
for rnd in range(6):
    for g in (1, 0):
        ley.ley_set_option("graphs", g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            ley.ley_sort(x, out, n)
        e1.record()
        torch.cuda.synchronize()
        res[g].append(e0.elapsed_time(e1) / 3)
print(n, "graphs", [round(v, 3) for v in res[1]], "direct", [round(v, 3) for v in res[0]],
      "median", round(statistics.median(res[1]), 3), round(statistics.median(res[0]), 3), flush=True)
