"""Drive mbt_gv (tools/mb_tma.cu): random 100-B record gather by bulk copy / tensor box / cp.async.

usage: python tools/mb_gv.py [n] [--once]
"""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmb_tma.so"))
lib.mbt_gv_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
n = int(float(sys.argv[1])) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 100_000_000
once = "--once" in sys.argv
g = torch.Generator(device="cuda")
g.manual_seed(0)
x = torch.randint(0, 256, (n * 128,), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
perm = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
s = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count
NAMES = ["bulk112", "tensor", "cpasync64", "cpasync", "bulk+pf2", "bulk+pf4", "bulk+pf8", "bulk128al"]
for mode, promo in [(int(m), 0) for m in os.environ.get("GV_MODES", "0,4,5,6").split(",")]:
    for stages, occ in ((2, 3), (3, 2), (4, 1), (1, 6)):
        args = (mode, stages, promo, x.data_ptr(), out.data_ptr(), perm.data_ptr(), n, sms * occ, s)
        rc = lib.mbt_gv_run(*args)
        assert rc == 0, rc
        torch.cuda.synchronize()
        ms = float("nan")
        if not once:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                lib.mbt_gv_run(*args)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
        o = out.view(n, 100)
        idx = torch.randint(0, n, (4096,), device="cuda", generator=g)
        ok = mode == 7 or torch.equal(o[idx], x[: n * 100].view(n, 100)[perm[idx].long()])
        print(f"{NAMES[mode]:10s} promo={promo:3d} stages={stages} ctas/sm={occ}  {ms:7.3f} ms  "
              f"{200 * n / ms / 1e6:6.0f} rec-r+w GB/s  {'ok' if ok else 'MISMATCH'}", flush=True)
