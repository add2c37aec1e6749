import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import gen, oracle
import paper_1909_08006_b200 as ley
for n, dist in [(31, "uniform"), (5, "uniform"), (4097, "uniform"), (300007, "uniform")]:
    recs = gen.records(n, seed=n, dist=dist)
    x = torch.from_numpy(recs).cuda(); out = torch.empty_like(x); perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ley.ley_sort_perm(x, out, perm, n)
    torch.cuda.synchronize()
    p = perm.cpu().numpy().view(np.uint32)
    exp, ep = oracle.sort(recs)
    o = out.cpu().numpy().reshape(-1, 100)
    bad = np.nonzero((o != exp.reshape(-1, 100)).any(axis=1))[0]
    print(n, "perm ok" if np.array_equal(p, ep) else "perm BAD", "bad recs", bad[:10].tolist())
    if not np.array_equal(p, ep):
        d = np.nonzero(p != ep)[0]
        print("  perm diff at", d[:10].tolist(), "gpu", p[d[:10]].tolist(), "exp", ep[d[:10]].tolist())
    if len(bad):
        j = bad[0]
        g = o[j]; e = exp.reshape(-1,100)[j]
        print("  byte diff positions", np.nonzero(g != e)[0].tolist()[:20])
