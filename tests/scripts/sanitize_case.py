"""Small sorts covering every kernel tier, recursion, the external path, the streaming path and the dist
loopback, each checked against the oracle — the workload for compute-sanitizer runs (one tool per run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import gen, oracle
import paper_1909_08006_b200 as ley

def check(recs, out, what):
    exp, _ = oracle.sort(recs)
    ok = np.array_equal(out, exp)
    print(what, "ok" if ok else "MISMATCH", flush=True)
    assert ok

for n, dist in [(5, "uniform"), (4097, "uniform"), (200_003, "uniform"), (200_003, "prefix2"),
                (120_001, "tiny_alphabet"), (150_001, "skewed"), (60_000, "all_equal")]:
    recs = gen.records(n, seed=7, dist=dist)
    x = torch.from_numpy(recs).cuda(); out = torch.empty_like(x)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ley.ley_sort_perm(x, out, perm, n); torch.cuda.synchronize()
    check(recs, out.cpu().numpy(), f"internal {dist} {n}")
# forced tiers
for kv in (dict(smem_tier_max=600), dict(kd_digit_bits=0), dict(warp_tier_max=4, kd_insert_max=1)):
    for k, v in kv.items(): ley.ley_set_option(k, v)
    recs = gen.records(70_001, seed=3, dist="skewed")
    x = torch.from_numpy(recs).cuda(); out = torch.empty_like(x)
    ley.ley_sort(x, out, 70_001); torch.cuda.synchronize()
    check(recs, out.cpu().numpy(), f"forced {kv}")
    for k in kv: ley.ley_set_option(k, {"smem_tier_max": 16384, "kd_digit_bits": 12, "warp_tier_max": 32, "kd_insert_max": 16}[k])
# external + streaming (pinned host)
recs = gen.records(300_000, seed=9, dist="uniform")
x = torch.from_numpy(recs).pin_memory(); out = torch.empty_like(x).pin_memory()
ley.ley_sort(x, out, 300_000, device_budget_bytes=12 << 20)
check(recs, out.numpy(), "external")
out2 = torch.empty_like(x).pin_memory()
ley.ley_sort_submit(x, out2, 300_000); ley.ley_sort_drain()
check(recs, out2.numpy(), "streaming")
# dist loopback G = 3
import ctypes
G, n = 3, 90_001
recs = gen.records(n, seed=11, dist="skewed")
bounds = [0, 30_000, 60_000, n]
ins = [torch.from_numpy(recs[bounds[i] * 100:bounds[i + 1] * 100].copy()).cuda() for i in range(G)]
outs = [torch.empty(n * 100, dtype=torch.uint8, device="cuda") for _ in range(G)]
res = ley.ley_sort_dist_loopback([t.data_ptr() for t in ins], [bounds[i + 1] - bounds[i] for i in range(G)],
                                 [t.data_ptr() for t in outs], [n] * G)
torch.cuda.synchronize()
cat = np.concatenate([outs[i][: res[i][0] * 100].cpu().numpy() for i in range(G)])
check(recs, cat, "dist loopback")
print("ALL OK")
