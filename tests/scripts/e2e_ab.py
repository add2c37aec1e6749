"""A/B of the streaming host sort's copy layout (option pipe_split): C2-sized pinned host in/out, 16 calls
through ley_sort_submit, CUDA-event time per call. usage: e2e_ab.py [n] [calls]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import gen
import oracle
import paper_1909_08006_b200 as ley
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 16
d = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
gen.records_cuda(d.data_ptr(), n, 1, "uniform")
hin = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
hin.copy_(d)
del d
torch.cuda.empty_cache()
hout = torch.empty_like(hin).pin_memory()
s = torch.cuda.current_stream()
for split in (1, 2, 3, 4, 2, 4):
    ley.ley_set_option("pipe_split", split)
    ley.ley_sort_submit(hin, hout, n)
    ley.ley_sort_drain()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(calls):
        ley.ley_sort_submit(hin, hout, n, stream=s)
    ley.ley_sort_drain()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / calls
    print(f"pipe_split={split}: {ms:.1f} ms/call = {n * 100 / ms / 1e6:.1f} GB/s", flush=True)
ley.ley_set_option("pipe_split", 2)
sl = hin[: 1_000_000 * 100].numpy()
print("sorted ok", oracle.is_sorted(hout.numpy()[: 100 * 1000]))
