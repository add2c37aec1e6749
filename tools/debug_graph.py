"""Graph-capture debugging: small sorts with graphs on/off, default vs torch streams; prints the library error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1909_08006_b200 as ley

for n in (1000, 1_000_000, 10_000_000):
    x = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
    gen.records_cuda(x.data_ptr(), n, 1, "uniform")
    out = torch.empty_like(x)
    for g in (1, 0):
        ley.ley_set_option("graphs", g)
        for stream in (None, torch.cuda.current_stream(), torch.cuda.Stream()):
            for rep in range(2):
                st = ley.ley_sort(x, out, n, stream=stream, raise_on_error=False)
                torch.cuda.synchronize()
                print(n, "graphs", g, "stream", "none" if stream is None else stream.cuda_stream, "rep", rep, "st", st,
                      ley.ley_last_error() if st else "", flush=True)
