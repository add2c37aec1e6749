"""Randomised parity stress (GPU): random sizes, distributions and library options, every output compared
with the CPU oracle byte for byte (records and permutation). For races the fixed test cases might miss
(tier overlap under PDL, dynamic bucket claims, stream-ordered calls back to back).

usage: python tests/scripts/stress.py [iterations] [seed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import gen
import oracle
import paper_1909_08006_b200 as ley

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
DISTS = ["uniform", "skewed", "all_equal", "three_keys", "sorted", "reverse", "prefix2", "byte9", "ascii",
         "tiny_alphabet"]
OPTS = {"pdl": [0, 1, 2, 3], "kd_claim": [0, 1], "async": [0, 1], "kd_ws": [0, 1], "graphs": [0, 1],
        "smem_tier_max": [600, 16384], "warp_tier_max": [4, 32]}
defaults = {k: ley.ley_get_option(k) for k in OPTS}
bad = 0
for it in range(iters):
    n = int(rng.choice([1, 7, 33, 513, 4097, 20000, 70001, 150001, 300007]))
    d = str(rng.choice(DISTS))
    opts = {k: int(rng.choice(v)) for k, v in OPTS.items()}
    for k, v in opts.items():
        ley.ley_set_option(k, v)
    recs = gen.records(n, seed=int(rng.integers(1 << 30)), dist=d)
    x = torch.from_numpy(recs).cuda()
    outs = []
    for rep in range(2):  # two calls back to back on the same stream (stream-ordered when async)
        out = torch.empty_like(x)
        perm = torch.empty(n, dtype=torch.int32, device="cuda")
        ley.ley_sort_perm(x, out, perm, n)
        outs.append((out, perm))
    torch.cuda.synchronize()
    exp, eperm = oracle.sort(recs)
    for out, perm in outs:
        ok = np.array_equal(out.cpu().numpy(), exp) and np.array_equal(perm.cpu().numpy().view(np.uint32), eperm)
        if not ok:
            bad += 1
            print("MISMATCH", it, n, d, opts, flush=True)
    for k, v in defaults.items():
        ley.ley_set_option(k, v)
print(f"stress: {iters} cases, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
