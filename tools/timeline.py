"""Live kernel timeline of one ley_sort call (CUPTI activity records through torch.profiler): start offset,
duration and gap to the previous kernel for every kernel the call launches — level 1 from its CUDA graph
included — to see where a small sort's time goes (launch gaps, empty tiers, host syncs).

usage: python tools/timeline.py N [DIST] [opt=v ...] [--flush]   (--flush: write 512 MB before the call: L2 cold)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import gen
import paper_1909_08006_b200 as ley

n = int(float(sys.argv[1]))
dist = sys.argv[2] if len(sys.argv) > 2 and "=" not in sys.argv[2] else "uniform"
flush = "--flush" in sys.argv
for kv in sys.argv[2:]:
    if "=" in kv:
        k, v = kv.split("=")
        ley.ley_set_option(k, int(v))
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(x.data_ptr(), n, 1, dist)
out = torch.empty_like(x)
for _ in range(5):
    ley.ley_sort(x, out, n)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    ley.ley_sort(x, out, n)
torch.cuda.synchronize()
print(f"host wall per call: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms")
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(20):
    if flush:
        junk.fill_(1)
    e0.record()
    ley.ley_sort(x, out, n)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"event-timed per call{' (L2 flushed before each)' if flush else ''}: median {ts[10]:.3f} ms, min {ts[0]:.3f}")
if flush:
    junk.fill_(1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ley.ley_sort(x, out, n)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
last = ev
base = last[0].time_range.start
prev_end = base
print(f"{'kernel':60s} {'start':>8s} {'dur':>8s} {'gap':>7s}  (us)")
for e in last:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    print(f"{e.name[:60]:60s} {s - base:8.1f} {d:8.1f} {s - prev_end:7.1f}")
    prev_end = e.time_range.end
print(f"span first start -> last end: {prev_end - base:.1f} us, kernels {len(last)}, sum of durations "
      f"{sum(e.time_range.end - e.time_range.start for e in last):.1f} us")
