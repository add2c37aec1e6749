"""Drive tools/mb_mem.cu: time 100-B-record gather vs scatter and friends on one B200 (CUDA events).

usage: python tools/mb_mem.py [n] [case ...]      (build: see tools/mb_build.sh)
"""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmb_mem.so"))
lib.mb_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
only = set(sys.argv[2:])
dev = "cuda"
torch.manual_seed(0)
x = torch.randint(0, 256, (n * 100,), dtype=torch.uint8, device=dev)
out = torch.empty_like(x)
idx_out = torch.empty(n, dtype=torch.int32, device=dev)
s = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count


def inverse(p):
    r = torch.empty_like(p)
    r[p.long()] = torch.arange(n, dtype=torch.int32, device=dev)
    return r


def win_perm(w):
    # random permutation inside consecutive windows of w records
    keys = torch.arange(n, device=dev, dtype=torch.int64) // w * 4 + 0
    r = torch.rand(n, device=dev, dtype=torch.float64)
    o = torch.argsort(keys.double() * 2 + r)
    return o.to(torch.int32)


def bucket_perm(bits):
    d = torch.randint(0, 1 << bits, (n,), device=dev, dtype=torch.int32)
    _, p = torch.sort(d, stable=True)
    return p.to(torch.int32)


def t(which, idx, grid, reps=3):
    ip = idx.data_ptr() if idx is not None else 0
    lib.mb_run(which, x.data_ptr(), out.data_ptr(), ip, idx_out.data_ptr(), n, grid, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        rc = lib.mb_run(which, x.data_ptr(), out.data_ptr(), ip, idx_out.data_ptr(), n, grid, s)
        assert rc == 0, rc
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rep(name, ms, bytes_per_rec):
    print(f"{name:28s} {ms:8.3f} ms  {bytes_per_rec * n / ms / 1e6:8.0f} GB/s at {bytes_per_rec} B/rec "
          f"({100 * n / ms / 1e6:7.0f} rec-GB/s)", flush=True)


g = sms * 8
cases = {}
perm = torch.randperm(n, device=dev).to(torch.int32)
rank = inverse(perm)
cases["copy"] = lambda: rep("copy", t(4, None, sms * 16), 200)
cases["keys"] = lambda: rep("keys (12 B loads)", t(3, None, sms * 16), 12)
cases["gather"] = lambda: rep("gather random", t(0, perm, g), 204)
cases["scatter"] = lambda: rep("scatter random", t(1, rank, g), 204)
cases["scatter_idx"] = lambda: rep("idx scatter random", t(2, perm, sms * 16), 8)
for name, fn in cases.items():
    if not only or name in only:
        fn()
for bits in (8, 12, 16):
    if only and f"b{bits}" not in only:
        continue
    pb = bucket_perm(bits)
    rep(f"gather stable-bucket{bits}", t(0, pb, g), 204)
    rep(f"scatter stable-bucket{bits}", t(1, inverse(pb), g), 204)
    del pb
for w in (24_576, 393_216, 1_572_864):
    if only and f"w{w}" not in only:
        continue
    pw = win_perm(w)
    rep(f"gather window {w * 100 / 1e6:.1f}MB", t(0, pw, g), 204)
    rep(f"scatter window {w * 100 / 1e6:.1f}MB", t(1, inverse(pw), g), 204)
    del pw

# L2-reuse study: which = 10 + mode + 4 * chunk_groups (mode bit0 L1 loads, bit1 blocked CTA chunks)
if "l2" in only:
    for w in (32, 256, 4096, 24_576):
        pw = win_perm(w)
        for mode in (0, 1):
            rep(f"gather2 m{mode} window {w}", t(10 + mode, pw, g), 204)
        if w >= 256:
            for mode in (2, 3):
                rep(f"gather2 m{mode} blocked window {w}", t(10 + mode + 4 * (w // 32), pw, g), 204)
        del pw

if "g3" in only:
    for grid_mult in (4, 8):
        rep(f"gather cp.async x{grid_mult}/SM", t(0, perm, sms * grid_mult), 204)
    for grid_mult in (2, 4, 6, 8):
        rep(f"gather reg x{grid_mult}/SM", t(5, perm, sms * grid_mult), 204)
    rep("gather bulk S2 x3/SM", t(6, perm, sms * 3), 204)
    rep("gather bulk S2 x2/SM", t(6, perm, sms * 2), 204)
    rep("gather bulk S3 x2/SM", t(8, perm, sms * 2), 204)
    rep("gather bulk S4 x1/SM", t(7, perm, sms * 1), 204)

if "g4" in only:
    rep("gather cp.async x8/SM", t(0, perm, sms * 8), 204)
    rep("gather bulk S2 x3/SM", t(6, perm, sms * 3), 204)
    # TMA-store variant: smem per CTA = 8 x (S x 3584 + 6400)
    for st, mults in ((1, (2, 4)), (2, (2, 3)), (3, (2,))):
        for m in mults:
            rep(f"gather tma S{st} x{m}/SM", t(19 + st, perm, sms * m), 204)
    # correctness of the tma variant: compare with the plain gather
    t(0, perm, sms * 8, reps=1); ref = out.clone()
    t(21, perm, sms * 2, reps=1)
    print("tma variant matches:", bool(torch.equal(ref, out)))
