"""Drive tools/mb_fetch.cu: time the key read and the random record gather under each L2 fetch granularity
and load qualifier. DRAM bytes come from ncu over the same command (tools/gpu_fetch.sh).

usage: python tools/mb_fetch.py FETCH_BYTES [n] [--once]     (FETCH_BYTES -1 = leave the device default)
"""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmb_fetch.so"))
lib.mbf_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p]

fetch = int(sys.argv[1])
n = int(float(sys.argv[2])) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 100_000_000
once = "--once" in sys.argv
dev = "cuda"
torch.cuda.init()
rc = lib.mbf_set_fetch(fetch)
print(f"# set fetch {fetch}: rc {rc}; device reports {lib.mbf_get_fetch()} B", flush=True)
g = torch.Generator(device=dev)
g.manual_seed(0)
x = torch.randint(0, 256, (n * 100 + 256,), dtype=torch.uint8, device=dev, generator=g)
out = torch.empty_like(x)
sink = torch.zeros(4, dtype=torch.int32, device=dev)
perm = torch.randperm(n, device=dev, generator=g).to(torch.int32)
s = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count
MODES = ["ld", "ld.cg", "ld.nc.noL1", "ld.L2::64B", "ld.L2::128B"]


def t(which, mode, grid, extra=0):
    args = (which, mode, x.data_ptr(), out.data_ptr(), perm.data_ptr(), sink.data_ptr(), n, grid, extra, s)
    assert lib.mbf_run(*args) == 0
    if once:
        torch.cuda.synchronize()
        return float("nan")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        assert lib.mbf_run(*args) == 0
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3


def rep(name, ms, useful_bytes):
    print(f"fetch={fetch:4d} {name:34s} {ms:8.3f} ms  useful {useful_bytes / ms / 1e6:8.0f} GB/s", flush=True)


rep("copy", t(3, 0, sms * 16), 200 * n)
for m in range(5):
    rep(f"keys 12B/rec [{MODES[m]}]", t(0, m, sms * 16), 12 * n)
for m in range(5):
    rep(f"gather 7x16B win [{MODES[m]}]", t(1, m, sms * 8), 200 * n)
for m in (0, 1, 2):
    rep(f"gather exact sectors [{MODES[m]}]", t(2, m, sms * 8), 200 * n)
for stride in (64, 128):
    for m in (0, 1):
        rep(f"probe 4B per {stride}B [{MODES[m]}]", t(4, m, sms * 16, stride), 4 * (100 * n // stride))
