"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and compare with the oracle."""
from __future__ import annotations

import numpy as np
import torch

import gen
import oracle
import paper_1909_08006_b200 as ley


def to_device(recs: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(recs)).cuda()


def gpu_sort(recs: np.ndarray, with_perm: bool = True, budget: int = 0):
    """ley_sort_perm on device copies of `recs`; returns (out, perm) as numpy."""
    n = recs.size // 100
    x = to_device(recs)
    out = torch.empty_like(x)
    if with_perm:
        perm = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        ley.ley_sort_perm(x, out, perm, n, device_budget_bytes=budget)
        torch.cuda.synchronize()
        return out.cpu().numpy(), perm[:n].cpu().numpy().view(np.uint32)
    ley.ley_sort(x, out, n, device_budget_bytes=budget)
    torch.cuda.synchronize()
    return out.cpu().numpy(), None


def assert_parity(recs: np.ndarray, out: np.ndarray, perm: np.ndarray | None = None):
    """Byte-exact equality with the oracle (and its permutation when given)."""
    exp, eperm = oracle.sort(recs)
    if not np.array_equal(out, exp):
        a, b = out.reshape(-1, 100), exp.reshape(-1, 100)
        bad = np.nonzero((a != b).any(axis=1))[0]
        raise AssertionError(f"{bad.size} of {a.shape[0]} records differ; first at {bad[:5].tolist()}")
    if perm is not None:
        assert np.array_equal(perm, eperm), "perm differs from the oracle's"


class Options:
    """Context manager that sets library options and restores the defaults."""

    def __init__(self, **kv):
        self.kv = kv
        self.old = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = ley.ley_get_option(k)
            ley.ley_set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            ley.ley_set_option(k, v)


def device_records(n: int, seed: int, dist="uniform") -> torch.Tensor:
    x = torch.empty(max(n, 1) * 100, dtype=torch.uint8, device="cuda")
    if n:
        gen.records_cuda(x.data_ptr(), n, seed, dist, stream=torch.cuda.current_stream().cuda_stream)
    return x[: n * 100]
