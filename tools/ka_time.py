"""Time K-a alone (ley_test_tile_sort) on device-resident synthetic records: uniform vs skewed, both forms."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
T = -(-n // 4096)
k1 = torch.empty(n, dtype=torch.int64, device="cuda"); w = torch.empty(n, dtype=torch.int32, device="cuda")
cnt = torch.empty(256 * T, dtype=torch.int32, device="cuda"); lo = torch.empty(T * 256, dtype=torch.int32, device="cuda")
h = torch.empty(65536, dtype=torch.int32, device="cuda")
x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
for dist, seed in (("uniform", 1), ("skewed", 2)):
    gen.records_cuda(x.data_ptr(), n, seed, dist)
    for form in (1, 0):
        ley.ley_test_tile_sort(x, n, k1, w, cnt, lo, h, stream_form=form)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ley.ley_test_tile_sort(x, n, k1, w, cnt, lo, h, stream_form=form)
        e1.record(); torch.cuda.synchronize()
        print(os.path.basename(os.environ.get("LEY_LIBRARY_OVERRIDE", "default")), dist, "form", form,
              f"{e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
