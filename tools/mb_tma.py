"""Drive tools/mb_tma.cu: key fetch and record gather by TMA tensor copies under each L2 promotion.

usage: python tools/mb_tma.py [n] [--once]   (bytes from ncu over the same command: tools/gpu_fetch2.sh)
"""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmb_tma.so"))
lib.mbt_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
n = int(float(sys.argv[1])) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 100_000_000
once = "--once" in sys.argv
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(0)
x = torch.randint(0, 256, (n * 100,), dtype=torch.uint8, device=dev, generator=g)
out = torch.empty_like(x)
sink = torch.zeros(4, dtype=torch.int32, device=dev)
perm = torch.randperm(n, device=dev, generator=g).to(torch.int32)
s = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count


def t(which, p, grid):
    args = (which, p, x.data_ptr(), out.data_ptr(), perm.data_ptr(), sink.data_ptr(), n, grid, s)
    rc = lib.mbt_run(*args)
    assert rc == 0, rc
    torch.cuda.synchronize()
    if once:
        return float("nan")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        assert lib.mbt_run(*args) == 0
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3


def check_gather():
    o = out.view(n, 100)
    idx = torch.randint(0, n, (4096,), device=dev, generator=g)
    ok = torch.equal(o[idx], x.view(n, 100)[perm[idx].long()])
    print(f"# gather check: {'ok' if ok else 'MISMATCH'}", flush=True)


for p in (0, 64, 128):
    for occ in (1, 2):
        ms = t(0, p, sms * occ)
        print(f"keys  promo={p:3d} grid={occ}x  {ms:8.3f} ms  {12 * n / ms / 1e6:7.0f} GB/s useful", flush=True)
for p in (0, 64, 128):
    for which, occ in ((1, 3), (2, 2), (3, 1)):
        out.zero_()
        ms = t(which, p, sms * occ)
        print(f"gather promo={p:3d} stages={which + 1} grid={occ}x  {ms:8.3f} ms  {200 * n / ms / 1e6:7.0f} GB/s rec r+w",
              flush=True)
        check_gather()
