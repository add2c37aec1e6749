"""Host-link bandwidth on this box: pinned H2D alone, D2H alone, and both at once (two streams), for a
few chunk sizes. The external path and the streaming e2e are bound by these numbers."""
import torch

GB = 1e9
for chunk_mb in (1, 4, 16, 64, 512):
    n = chunk_mb << 20
    reps = max(2, (8 << 30) // n)
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run(h2d, d2h):
        torch.cuda.synchronize()
        e0.record()
        s1.wait_event(e0); s2.wait_event(e0)
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s1):
                    d_a.copy_(h_in, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    t1 = run(True, False); t2 = run(False, True); t3 = run(True, True)
    b = reps * n / GB
    print(f"chunk {chunk_mb:5d} MB: H2D {b / t1:6.1f} GB/s  D2H {b / t2:6.1f} GB/s  both {b / t3:6.1f} + {b / t3:6.1f} GB/s",
          flush=True)

# H2D from cudaHostRegister'ed (mapped) memory, and many small copies back to back (external merge pattern)
import numpy as np
cr = torch.cuda.cudart()
n = 256 << 20
a = np.empty(n, dtype=np.uint8); a[:] = 1
cr.cudaHostRegister(a.ctypes.data, n, 2)  # cudaHostRegisterMapped
d = torch.empty(n, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
src = torch.from_numpy(a)
for piece in (4 << 20, 64 << 20):
    torch.cuda.synchronize(); e0.record()
    for rep in range(8):
        for o in range(0, n, piece):
            d[o:o + piece].copy_(src[o:o + piece], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"registered-mapped H2D in {piece >> 20} MB pieces: {8 * n / 1e9 / (e0.elapsed_time(e1) / 1e3):.1f} GB/s")
