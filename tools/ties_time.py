"""Long keys (key_bytes 20) when the 10-byte prefixes tie in many small groups: total time and the
tie-group stage, device-resident input. Groups of the given sizes (cycled), distinct prefixes.
Run: gpurun -- 'python tools/ties_time.py'"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_08006_b200 as ley  # noqa: E402

for n, sizes in ((20_000_000, [2]), (20_000_000, [2, 3, 5, 8]), (20_000_000, [67]), (20_000_000, [500]),
                 (20_000_000, [1])):
    rng = np.random.default_rng(1)
    r = rng.integers(0, 256, size=(n, 100), dtype=np.uint8)
    gid = np.repeat(np.arange(n, dtype=np.uint64), np.resize(np.asarray(sizes), n))[:n]
    gid = gid[rng.permutation(n)] * np.uint64(2654435761) + np.uint64(12345)
    r[:, 0:2] = 7
    for b in range(8):
        r[:, 9 - b] = (gid >> np.uint64(8 * b)) & np.uint64(0xFF)
    x = torch.from_numpy(r.reshape(-1)).cuda()
    out = torch.empty_like(x)
    for _ in range(2):
        ley.ley_sort(x, out, n, key_bytes=20)
    ley.ley_set_option("profile", 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    reps = 5
    stages = {}
    for _ in range(reps):
        ley.ley_sort(x, out, n, key_bytes=20)
        for name, ms in ley.ley_stage_times()[0]:
            stages[name] = stages.get(name, 0) + ms / reps
    e1.record()
    torch.cuda.synchronize()
    ley.ley_set_option("profile", 0)
    hybrid = e0.elapsed_time(e1) / reps
    ley.ley_set_option("key_hybrid", 0)
    ley.ley_sort(x, out, n, key_bytes=20)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        ley.ley_sort(x, out, n, key_bytes=20)
    e1.record()
    torch.cuda.synchronize()
    ley.ley_set_option("key_hybrid", 1)
    lsd = e0.elapsed_time(e1) / reps
    print(f"n {n:,} group sizes {sizes}: {hybrid:.2f} ms per sort; "
          f"tie groups {stages.get('tie groups', 0):.2f} ms; K-de {stages.get('K-de sort+gather', 0):.2f} ms", flush=True)
    print(f"   (LSD window passes instead of the hybrid: {lsd:.2f} ms)")
