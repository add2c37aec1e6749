"""Host-link microbenchmark for the external merge (DESIGN.md §9 next 5): H2D of a
partition as R separate run slices (the merge's current pattern) vs one contiguous copy, with and without a
concurrent D2H stream, from pinned host memory.

usage: python tools/mb_h2d_slices.py [total_GB] [R]
"""
import sys
import time

import torch

GB = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
R = int(sys.argv[2]) if len(sys.argv) > 2 else 63
total = int(GB * (1 << 30))
part = 300 << 20  # bytes per partition (C5 scaled: ~3M records)
parts = max(1, total // part)
host = torch.empty(parts * part, dtype=torch.uint8).pin_memory()
hout = torch.empty(parts * part, dtype=torch.uint8).pin_memory()
dev = torch.empty(2 * part, dtype=torch.uint8, device="cuda")
dout = torch.empty(part, dtype=torch.uint8, device="cuda")
h2d = torch.cuda.Stream()
d2h = torch.cuda.Stream()
sl = part // R


def run(mode, with_d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for p in range(parts):
        dst = dev[(p & 1) * part:(p & 1) * part + part]
        with torch.cuda.stream(h2d):
            if mode == "slices":
                for r in range(R):  # slice r of partition p sits in run r's region: stride = parts * sl
                    src_off = (r * parts + p) * sl
                    dst[r * sl:(r + 1) * sl].copy_(host[src_off:src_off + sl], non_blocking=True)
            else:
                dst.copy_(host[p * part:(p + 1) * part], non_blocking=True)
        if with_d2h:
            with torch.cuda.stream(d2h):
                hout[p * part:(p + 1) * part].copy_(dout, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{mode:7s} d2h={with_d2h!s:5s} parts {parts} x {part >> 20} MB ({R} slices of {sl / 2**20:.1f} MB): "
          f"{dt * 1e3:8.1f} ms  H2D {parts * part / dt / 1e9:6.1f} GB/s", flush=True)


def run_d2h(mode, with_h2d):
    """The mirror image: D2H of each partition-sized device buffer as R slices (partition-major run
    writing) or whole, with an optional concurrent whole-buffer H2D stream."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for p in range(parts):
        src = dev[(p & 1) * part:(p & 1) * part + part]
        with torch.cuda.stream(d2h):
            if mode == "slices":
                for r in range(R):
                    dst_off = (r * parts + p) * sl
                    hout[dst_off:dst_off + sl].copy_(src[r * sl:(r + 1) * sl], non_blocking=True)
            else:
                hout[p * part:(p + 1) * part].copy_(src, non_blocking=True)
        if with_h2d:
            with torch.cuda.stream(h2d):
                dout.copy_(host[p * part:(p + 1) * part], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"D2H {mode:7s} h2d={with_h2d!s:5s}: {dt * 1e3:8.1f} ms  D2H {parts * part / dt / 1e9:6.1f} GB/s", flush=True)


for _ in range(2):
    for mode in ("slices", "whole"):
        for wd in (False, True):
            run(mode, wd)
    for mode in ("slices", "whole"):
        for wd in (False, True):
            run_d2h(mode, wd)
