"""Zero-copy host link throughput: a grid-stride 16-B copy kernel (tools/mb_mem.cu mb_copy) reading or
writing pinned host memory directly, alone and with both directions at once, versus the copy engines."""
import ctypes, os
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmb_mem.so"))
lib.mb_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
nrec = 20_000_000  # 2 GB
B = nrec * 100
h_in = torch.empty(B, dtype=torch.uint8).pin_memory(); h_in.fill_(3)
h_out = torch.empty(B, dtype=torch.uint8).pin_memory()
d_a = torch.empty(B, dtype=torch.uint8, device="cuda")
d_b = torch.empty(B, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def run(h2d, d2h, grid, engine=False, reps=3, mixed=False):
    torch.cuda.synchronize(); e0.record(); s1.wait_event(e0); s2.wait_event(e0)
    for _ in range(reps):
        if h2d:
            if engine:
                with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
            else:
                lib.mb_run(4, h_in.data_ptr(), d_a.data_ptr(), None, None, nrec, grid, s1.cuda_stream)
        if d2h:
            if engine or mixed:
                with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
            else:
                lib.mb_run(4, d_b.data_ptr(), h_out.data_ptr(), None, None, nrec, grid, s2.cuda_stream)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    return reps * B / 1e9 / (e0.elapsed_time(e1) / 1e3)

print(f"engines: H2D {run(1,0,0,True):.1f}  D2H {run(0,1,0,True):.1f}  both {run(1,1,0,True):.1f} each GB/s")
for grid in (8, 16, 32, 64, 148):
    print(f"kernel grid {grid:4d}: H2D {run(1,0,grid):.1f}  D2H {run(0,1,grid):.1f}  both {run(1,1,grid):.1f} each GB/s", flush=True)
for grid in (32, 64, 148):
    print(f"kernel H2D grid {grid} + engine D2H: both {run(1,1,grid,mixed=True):.1f} each GB/s", flush=True)
d_a.copy_(h_in); assert bool((d_a[:1000] == 3).all())
