import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
import gen, oracle
import paper_1909_08006_b200 as ley
n = int(sys.argv[1]); dist = sys.argv[2]; seed = int(sys.argv[3])
opts = dict(kv.split("=") for kv in sys.argv[4:])
for k, v in opts.items():
    ley.ley_set_option(k, int(v))
ley.ley_set_option("profile", 1)
recs = gen.records(n, seed=seed, dist=dist)
x = torch.from_numpy(recs).cuda(); out = torch.empty_like(x); perm = torch.empty(n, dtype=torch.int32, device="cuda")
t = time.time()
ley.ley_sort_perm(x, out, perm, n)
torch.cuda.synchronize()
print("sorted in", time.time() - t, ley.ley_stage_times())
exp, ep = oracle.sort(recs)
print("parity", np.array_equal(out.cpu().numpy(), exp), np.array_equal(perm.cpu().numpy().view(np.uint32), ep))
