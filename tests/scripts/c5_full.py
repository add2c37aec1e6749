"""Full-size C5 (BASELINE.json configs[4]): 6e8 x 100-B uniform records (60 GB, seed 4) in pinned host memory,
device budget 4 GiB; the external path (run generation + merge-path K-way merge) through ley_sort, timed with
CUDA events, then verified in digest mode: the order-dependent sequence digest of `out` equals the oracle's
sorted digest of `in` (oracle/oracle.cpp oracle_sorted_digest: the tuple sort of the 6e8 keys on the host).

Host memory: in 60 GB + out 60 GB + the library's run scratch 60 GB (pinned) = 180 GB of the box's 196 GB;
the scratch is released (ley_release_cache) before the oracle's 12 GB of tuples are built.

usage: python tests/scripts/c5_full.py [n] [steps] [--keyptr]   -> one JSON line (profiles/r02_c5_full*.json)
--keyptr: the key-pointer form of the external path (option ext_keyptr): runs of 16-byte
tuples (9.6 GB of host scratch instead of 60 GB), records gathered from the pinned input by ordinal.
"""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import gen
import oracle
import paper_1909_08006_b200 as ley

args = [a for a in sys.argv[1:] if not a.startswith("--")]
keyptr = "--keyptr" in sys.argv
n = int(float(args[0])) if len(args) > 0 else 600_000_000
steps = int(args[1]) if len(args) > 1 else 2
budget = 4 << 30
seed = 4


def free_gb():
    return subprocess.run(["free", "-g"], capture_output=True, text=True).stdout.splitlines()[1].split()[1:4]


res = {"config": f"C5 full: {n:,} x 100 B uniform, seed {seed}, pinned host in/out, device budget 4 GiB",
       "free_gb_start": free_gb(), "plan": ley.ley_plan_query(n, budget)}
t0 = time.time()
import numpy as np


def pinned(nbytes):
    """Page-locked host buffer of exactly nbytes (numpy + cudaHostRegister; torch's pinned allocator would
    round 60 GB up to a power of two)."""
    a = np.empty(nbytes, dtype=np.uint8)
    rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, nbytes, 2)  # cudaHostRegisterMapped
    assert int(rc) == 0, f"cudaHostRegister failed: {rc}"
    return a, torch.from_numpy(a)


xa, x = pinned(n * 100)
oa, out = pinned(n * 100)
stage = torch.empty(50_000_000 * 100, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for at in range(0, n, 50_000_000):
    m = min(50_000_000, n - at)
    gen.records_cuda(stage.data_ptr(), m, seed, "uniform", i0=at, stream=s.cuda_stream)
    x[at * 100:(at + m) * 100].copy_(stage[: m * 100])
del stage
torch.cuda.empty_cache()
res["setup_s"] = round(time.time() - t0, 1)
if keyptr:
    ley.ley_set_option("ext_keyptr", 1)
    res["config"] += " (key-pointer external form)"
ley.ley_sort(x, out, n, device_budget_bytes=budget, stream=s)  # warm: run scratch, streams
res["free_gb_after_warm"] = free_gb()
ley.ley_set_option("profile", 1)
times, stages = [], []
for _ in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ley.ley_sort(x, out, n, device_budget_bytes=budget, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
    stages.append({k: round(v, 1) for k, v in ley.ley_stage_times()[0]})
ley.ley_set_option("profile", 0)
cur, peak = ley.ley_device_bytes()
res.update({"ms_per_step": [round(t, 1) for t in times], "sorted_gb_s": round(n * 100 / (min(times) / 1e3) / 1e9, 2),
            "stages_ms": stages, "device_bytes_peak": peak, "device_budget_bytes": budget})
ley.ley_release_cache(-1)
t1 = time.time()
got = oracle.sequence_digest(oa)
exp = oracle.sorted_digest(xa)
res["verify"] = {"kind": "digest: sequence_digest(out) == oracle sorted_digest(in)", "equal": got == exp,
                 "seconds": round(time.time() - t1, 1), "cores": os.cpu_count()}
mh_in, mh_out = oracle.multiset_hash(xa), oracle.multiset_hash(oa)
res["verify"]["multiset_hash_equal"] = mh_in == mh_out
res["free_gb_end"] = free_gb()
print(json.dumps(res), flush=True)
