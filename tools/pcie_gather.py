"""Host-link cost of the key-pointer external path, measured rather than modelled.

That path would (1) bring only the keys to the device, (2) sort (key, ordinal) there, (3) gather the
payloads from pinned host in sorted order while streaming the output back. This measures its two host-link
phases with the tools/mb_mem.cu kernels on pinned host memory (zero-copy, UVA pointers):
  keys     mb_keys: 12 B (key + 2) of every 100-B record read in place     vs copy-engine H2D of the records
  gather   mb_gather: 100-B records at random host positions -> device      alone, and next to an engine D2H
and projects C5 (2e8 records) against the current external path (bench: 1022.7 ms).
Run: gpurun -- 'bash tools/mb_build.sh && python tools/pcie_gather.py'
"""
import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmb_mem.so"))
lib.mb_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
nrec = 20_000_000  # 2 GB of records
B = nrec * 100
h_in = torch.empty(B, dtype=torch.uint8).pin_memory()
h_in.fill_(3)
h_out = torch.empty(B, dtype=torch.uint8).pin_memory()
d_a = torch.empty(B, dtype=torch.uint8, device="cuda")
d_b = torch.empty(B, dtype=torch.uint8, device="cuda")
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
perm_rand = torch.randperm(nrec, device="cuda", dtype=torch.int64).to(torch.int32)
perm_seq = torch.arange(nrec, device="cuda", dtype=torch.int32)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn_h2d, d2h, reps=3):
    torch.cuda.synchronize()
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(reps):
        fn_h2d(s1)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps  # s per pass over the 2 GB


def engine_h2d(s):
    with torch.cuda.stream(s):
        d_a.copy_(h_in, non_blocking=True)


def gather(perm, grid, mode):
    return lambda s: lib.mb_run(mode, h_in.data_ptr(), d_a.data_ptr(), perm.data_ptr(), None, nrec, grid, s.cuda_stream)


def keys(grid):
    return lambda s: lib.mb_run(3, h_in.data_ptr(), None, None, sink.data_ptr(), nrec, grid, s.cuda_stream)


# gather kernels (tools/mb_mem.cu): 0 cp.async 16-B pieces, 5 16-B register loads, 6/7 cp.async.bulk
# 112-B windows with 2/4 stages, 21 bulk windows + bulk store
MODES = {0: "cp.async", 5: "ld.v4", 6: "bulk x2", 7: "bulk x4", 21: "bulk+store x2"}
gbs = lambda t: B / 1e9 / t
t_eng = timed(engine_h2d, False)
print(f"engine H2D records: {gbs(t_eng):.1f} GB/s ({t_eng * 1e9 / nrec:.2f} ns/record)")
t_keys_best, t_gather_best = t_eng, 1e9
for grid in (148, 296, 592):
    tk = timed(keys(grid), False)
    t_keys_best = min(t_keys_best, tk)
    print(f"grid {grid:4d}: keys in place {tk * 1e9 / nrec:.2f} ns/record", flush=True)
    for mode, name in MODES.items():
        ts = timed(gather(perm_seq, grid, mode), False)
        tr = timed(gather(perm_rand, grid, mode), False)
        trd = timed(gather(perm_rand, grid, mode), True)
        t_gather_best = min(t_gather_best, trd)
        print(f"   gather {name:14s} seq {gbs(ts):5.1f} GB/s, random {gbs(tr):5.1f} GB/s, "
              f"random + engine D2H {gbs(trd):5.1f} GB/s", flush=True)
n5 = 200_000_000
t_keys = t_keys_best * n5 / nrec
t_gather = t_gather_best * n5 / nrec
print(f"C5 projection (2e8 records, best of each): keys phase {t_keys * 1e3:.0f} ms + gather/D2H phase "
      f"{t_gather * 1e3:.0f} ms = {(t_keys + t_gather) * 1e3:.0f} ms (+ the device sort) vs 1022.7 ms for the "
      f"current external path")
d_a.copy_(h_in)
assert bool((d_a[:1000] == 3).all())
