"""Drive tools/mb_l2.cu: random gather within a W-record region, cold vs after an evict_last sequential read.

usage: python tools/mb_l2.py [--once]
"""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmb_l2.so"))
lib.l2_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                       ctypes.c_int, ctypes.c_void_p]
once = "--once" in sys.argv
N = 100_000_000
x = torch.randint(0, 256, (N * 100,), dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty(4_000_000 * 100, dtype=torch.uint8, device="cuda")
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count
for W in (131072, 400_000, 1_000_000, 2_000_000):
    base = 37_000_000
    reg = x[base * 100:(base + W) * 100]
    perm = torch.randperm(W, device="cuda").to(torch.int32)
    for warm in (0, 1):
        times = []
        for rep in range(1 if once else 3):
            flush.zero_()  # evict the region
            if warm:
                assert lib.l2_run(0, reg.data_ptr(), None, None, sink.data_ptr(), W, sms * 8, s) == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert lib.l2_run(1, reg.data_ptr(), out.data_ptr(), perm.data_ptr(), None, W, sms * 8, s) == 0
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = min(times)
        ok = torch.equal(out[:W * 100].view(W, 100)[:1000], reg.view(W, 100)[perm[:1000].long()])
        print(f"W={W:9d} ({W * 100 / 1e6:6.1f} MB) {'after evict_last read' if warm else 'cold               '}: gather "
              f"{ms * 1e3:8.1f} us = {W / ms / 1e6:6.2f} G rec/s {'ok' if ok else 'MISMATCH'}", flush=True)
