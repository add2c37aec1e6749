"""A/B of library options in one process: per option set, the mean per-stage times of ley_sort on a
device-resident synthetic workload, with an on-device sortedness + byte-sum check of the output.

usage: python tools/ab_opts.py N DIST 'name:opt=v,opt=v' ['name2:...' ...]      ('base:' = defaults)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1909_08006_b200 as ley

n = int(float(sys.argv[1]))
dist = sys.argv[2]
variants = sys.argv[3:] or ["base:"]
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 1, dist)
out = torch.empty_like(x)
step = 1 << 30
s_in = sum(int(x[i:i + step].sum(dtype=torch.int64)) for i in range(0, x.numel(), step))


def check():
    r = out.view(n, 100)
    ok = True
    for c0 in range(0, n - 1, 1 << 27):
        c1 = min(n, c0 + (1 << 27) + 1)
        kb = lambda j: r[c0:c1, j].to(torch.int64)
        h = (kb(0) << 24) | (kb(1) << 16) | (kb(2) << 8) | kb(3)
        m = (kb(4) << 24) | (kb(5) << 16) | (kb(6) << 8) | kb(7)
        lo = (kb(8) << 8) | kb(9)
        good = (h[1:] > h[:-1]) | ((h[1:] == h[:-1]) & ((m[1:] > m[:-1]) | ((m[1:] == m[:-1]) & (lo[1:] >= lo[:-1]))))
        ok = ok and bool(good.all())
    s_out = sum(int(out[i:i + step].sum(dtype=torch.int64)) for i in range(0, out.numel(), step))
    return ok and s_out == s_in


defaults = {}
for v in variants:
    name, _, spec = v.partition(":")
    opts = dict(kv.split("=") for kv in spec.split(",") if kv)
    for k, val in opts.items():
        defaults.setdefault(k, ley.ley_get_option(k))
        ley.ley_set_option(k, int(val))
    out.zero_()
    for _ in range(2):
        ley.ley_sort(x, out, n)
    ok = check()
    ley.ley_set_option("profile", 1)
    acc = {}
    tot = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ley.ley_sort(x, out, n)
        e1.record()
        torch.cuda.synchronize()
        tot.append(e0.elapsed_time(e1))
        for k, val in ley.ley_stage_times()[0]:
            acc.setdefault(k, []).append(val)
    ley.ley_set_option("profile", 0)
    plain = []
    for _ in range(5):  # without stage events (level 1 from its CUDA graph)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ley.ley_sort(x, out, n)
        e1.record()
        torch.cuda.synchronize()
        plain.append(e0.elapsed_time(e1))
    print(f"{name:14s} {dist} n={n} {'CHECK-OK' if ok else 'CHECK-FAILED'} plain {statistics.median(plain):.3f} ms "
          f"profiled {statistics.median(tot):.3f} ms",
          {k: round(statistics.mean(vv), 3) for k, vv in acc.items()}, flush=True)
    for k, val in defaults.items():
        ley.ley_set_option(k, val)
