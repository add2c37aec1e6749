"""Runtime behaviour around the hot path (SURVEY.md §8b conventions): concurrent callers on one device are
serialised by the library (every result still byte-exact), the caller's stream orders the work, and a
failed device allocation is reported (LEY_ERR_CUDA, stage-tagged) without poisoning later calls."""
import threading

import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu


def test_concurrent_callers_one_device(cuda_ok):
    """Six threads at once on one device: device-pointer sorts, staged host sorts, a resident-path sort and
    a streaming submit/drain, each on its own data. The library serialises them (per-device mutex, the
    pipeline's own lock) and every output equals the oracle's."""
    import paper_1909_08006_b200 as ley

    jobs = []
    for t in range(6):
        n = 120_001 + 7919 * t
        recs = gen.records(n, seed=200 + t, dist=("uniform", "skewed", "three_keys")[t % 3])
        jobs.append((t, n, recs, oracle.sort(recs)[0]))
    errors = []

    def work(t, n, recs, exp):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    if t in (0, 1):  # device pointers
                        x = torch.from_numpy(recs).cuda()
                        out = torch.empty_like(x)
                        ley.ley_sort(x, out, n, stream=s)
                        got = out.cpu().numpy()
                    elif t in (2, 3):  # staged host path
                        x = torch.from_numpy(recs).pin_memory()
                        out = torch.empty_like(x).pin_memory()
                        ley.ley_sort(x, out, n, stream=s)
                        got = out.numpy()
                    elif t == 4:  # resident host path (budget between resident and staged)
                        x = torch.from_numpy(recs).pin_memory()
                        out = torch.empty_like(x).pin_memory()
                        ley.ley_sort(x, out, n, device_budget_bytes=ley.ley_plan_query(n, 1)["resident_bytes"],
                                     stream=s)
                        got = out.numpy()
                    else:  # streaming submit
                        x = torch.from_numpy(recs).pin_memory()
                        out = torch.empty_like(x).pin_memory()
                        ley.ley_sort_submit(x, out, n, stream=s)
                        ley.ley_sort_drain()
                        got = out.numpy()
                    if not np.array_equal(got, exp):
                        errors.append(f"thread {t} rep {rep}: output differs")
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(f"thread {t}: {e!r}")

    th = [threading.Thread(target=work, args=j) for j in jobs]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errors, errors


def test_stream_ordering(cuda_ok):
    """ley_sort orders its work after what is already enqueued on the caller's stream: the input is
    produced by a kernel still running on that stream when the call is made."""
    import paper_1909_08006_b200 as ley

    n = 200_003
    recs = gen.records(n, seed=9, dist="skewed")
    src = torch.from_numpy(recs).cuda()
    s = torch.cuda.Stream()
    x = torch.empty_like(src)
    out = torch.empty_like(src)
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)  # ~tens of ms of spinning ahead of the copy on s
        x.copy_(src)
        ley.ley_sort(x, out, n, stream=s)
    s.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.sort(recs)[0])


def test_allocation_failure_is_reported_and_recoverable(cuda_ok):
    """With the device nearly full, a sort whose workspace cannot be allocated fails with LEY_ERR_CUDA and a
    stage-tagged message; after the memory is freed the same call succeeds and is exact."""
    import paper_1909_08006_b200 as ley

    n = 20_000_000  # 2 GB in + 2 GB out; the library's scratch ~0.6 GB more
    recs_dev = torch.empty(n * 100, dtype=torch.uint8, device="cuda")
    gen.records_cuda(recs_dev.data_ptr(), n, 3, "uniform")
    out = torch.empty_like(recs_dev)
    ley.ley_release_cache(-1)
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    hog = torch.empty(max(free - (64 << 20), 0), dtype=torch.uint8, device="cuda")  # leave ~64 MB
    try:
        st = ley.ley_sort(recs_dev, out, n, raise_on_error=False)
        assert st == ley.LEY_ERR_CUDA, st
        msg = ley.ley_last_error()
        assert msg and ":" in msg, msg
    finally:
        del hog
        torch.cuda.empty_cache()
    ley.ley_sort(recs_dev, out, n)
    sl = recs_dev[: 500_000 * 100].cpu().numpy()
    o2 = torch.empty(500_000 * 100, dtype=torch.uint8, device="cuda")
    ley.ley_sort(recs_dev[: 500_000 * 100], o2, 500_000)
    assert np.array_equal(o2.cpu().numpy(), oracle.sort(sl)[0])
    # the full output is certified by sortedness + multiset equality against the input
    h_in, h_out = recs_dev.cpu().numpy(), out.cpu().numpy()
    assert oracle.is_sorted(h_out)
    assert oracle.multiset_hash(h_in) == oracle.multiset_hash(h_out)
    ley.ley_release_cache(-1)
