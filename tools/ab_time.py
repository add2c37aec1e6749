"""Average per-stage times of ley_sort on a device-resident synthetic workload (A/B of library variants
via LEY_LIBRARY_OVERRIDE), plus a cheap on-device sanity check of the output (keys non-decreasing and
byte sum preserved) so a broken variant cannot report a time.

usage: python tools/ab_time.py [n] [dist] [steps] [seed]
"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
dist = sys.argv[2] if len(sys.argv) > 2 else "uniform"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 1
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, seed, dist)
out = torch.empty_like(x)
for _ in range(2):
    ley.ley_sort(x, out, n)


def check():
    r = out.view(n, 100)
    kb = lambda j: r[:, j].to(torch.int64)
    h = (kb(0) << 24) | (kb(1) << 16) | (kb(2) << 8) | kb(3)
    m = (kb(4) << 24) | (kb(5) << 16) | (kb(6) << 8) | kb(7)
    lo = (kb(8) << 8) | kb(9)
    ok = (h[1:] > h[:-1]) | ((h[1:] == h[:-1]) & ((m[1:] > m[:-1]) | ((m[1:] == m[:-1]) & (lo[1:] >= lo[:-1]))))
    good = bool(ok.all())
    step = 1 << 30
    s_in = sum(int(x[i:i + step].sum(dtype=torch.int64)) for i in range(0, x.numel(), step))
    s_out = sum(int(out[i:i + step].sum(dtype=torch.int64)) for i in range(0, out.numel(), step))
    return good and s_in == s_out


ok = check()
ley.ley_set_option("profile", 1)
acc = {}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    ley.ley_sort(x, out, n)
    for k, v in ley.ley_stage_times()[0]:
        acc.setdefault(k, []).append(v)
e1.record(); torch.cuda.synchronize()
tag = os.path.basename(os.environ.get("LEY_LIBRARY_OVERRIDE", "default"))
print(tag, dist, n, "CHECK-OK" if ok else "CHECK-FAILED", f"total {e0.elapsed_time(e1)/steps:.3f} ms",
      {k: round(statistics.mean(v), 3) for k, v in acc.items()}, flush=True)
