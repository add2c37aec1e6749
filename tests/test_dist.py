"""Multi-GPU key-range sort.

* -m gpu: the loopback transport runs the real G-rank algorithm (K-s0/K-s1/K-s2/K-p kernels, plans, local
  sort) on one B200, with K-p storing straight into every receiver's buffer (fused exchange, the
  kernels never wait on one another) or device copies standing in for the all-to-all; and the NCCL path
  itself at world size 1, including its exchange phase (symmetric window or send/recv to itself).
  Checks: concatenation of the ranks' outputs == oracle of the concatenated input; closed-form sizes
  n_out(r) = floor((r+1)N/G) - floor(rN/G) and offsets floor(rN/G) (exact splitters).
* -m "not gpu": two gloo processes run the host-side planning of the library (ley_dist_plan_splitters,
  ley_dist_bin_dest_counts, ley_dist_plan_exchange) around a numpy stand-in for the kernels and a real
  all-to-all, and must reproduce the oracle.
"""
import os
import socket

import numpy as np
import pytest

import gen
import oracle


def _closed_form(N, G):
    return [((r + 1) * N // G) - (r * N // G) for r in range(G)], [r * N // G for r in range(G)]


# ----------------------------------------------------------------------------------------- GPU
@pytest.fixture(params=[1, 0], ids=["fused", "alltoall"])
def exchange_mode(request):
    """dist_fused=1: K-p stores into the receivers' buffers; 0: send buffer + all-to-all-v."""
    import paper_1909_08006_b200 as ley

    ley.ley_set_option("dist_fused", request.param)
    yield request.param
    ley.ley_set_option("dist_fused", 1)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dist", ["uniform", "skewed", "all_equal", "tiny_alphabet", "sorted", "reverse"])
def test_loopback_matches_oracle(cuda_ok, exchange_mode, G, dist):
    import torch

    import paper_1909_08006_b200 as ley

    rng = np.random.default_rng(G * 7 + len(dist))
    N = 90_001
    cuts = np.sort(rng.integers(0, N, size=G - 1))
    n_local = np.diff(np.concatenate([[0], cuts, [N]])).tolist()
    if G > 2:
        n_local[1] += n_local[2]  # one empty rank
        n_local[2] = 0
    recs = gen.records(N, seed=51, dist=dist)
    ins, outs, caps = [], [], []
    at = 0
    for r in range(G):
        part = recs[at * 100:(at + n_local[r]) * 100]
        at += n_local[r]
        ins.append(torch.from_numpy(part.copy()).cuda() if n_local[r] else torch.empty(100, dtype=torch.uint8,
                                                                                       device="cuda"))
        cap = N // G + 2
        outs.append(torch.empty(cap * 100, dtype=torch.uint8, device="cuda"))
        caps.append(cap)
    res = ley.ley_sort_dist_loopback(ins, n_local, outs, caps)
    torch.cuda.synchronize()
    sizes, offs = _closed_form(N, G)
    assert [x[0] for x in res] == sizes
    assert [x[1] for x in res] == offs
    got = np.concatenate([outs[r][: res[r][0] * 100].cpu().numpy() for r in range(G)])
    exp, _ = oracle.sort(recs)
    assert np.array_equal(got, exp)


@pytest.mark.gpu
def test_loopback_tiny_and_capacity(cuda_ok, exchange_mode):
    import torch

    import paper_1909_08006_b200 as ley

    G, N = 8, 5  # fewer records than ranks
    recs = gen.records(N, seed=3)
    n_local = [1, 0, 2, 0, 0, 1, 1, 0]
    ins, outs, at = [], [], 0
    for r in range(G):
        ins.append(torch.from_numpy(recs[at * 100:(at + n_local[r]) * 100].copy()).cuda() if n_local[r]
                   else torch.empty(100, dtype=torch.uint8, device="cuda"))
        at += n_local[r]
        outs.append(torch.empty(200, dtype=torch.uint8, device="cuda"))
    res = ley.ley_sort_dist_loopback(ins, n_local, outs, [2] * G)
    sizes, offs = _closed_form(N, G)
    assert [x[0] for x in res] == sizes and [x[1] for x in res] == offs
    got = np.concatenate([outs[r][: res[r][0] * 100].cpu().numpy() for r in range(G)])
    assert np.array_equal(got, oracle.sort(recs)[0])
    # capacity error path
    with pytest.raises(ley.LeyendaError) as ei:
        ley.ley_sort_dist_loopback(ins, n_local, outs, [0] * G)
    assert ei.value.status == ley.LEY_ERR_CAPACITY


@pytest.mark.gpu
@pytest.mark.parametrize("exchange_g1", [0, 1], ids=["local", "exchange"])
def test_nccl_world_size_one(cuda_ok, exchange_mode, exchange_g1):
    """The NCCL path itself (communicator of one rank): equals ley_sort. With dist_exchange_g1 the rank
    also runs K-s0, K-p and the exchange: fused = ncclMemAlloc + symmetric window registration, the
    device-API peer-pointer table (its own entry is the local mapping), K-p storing into the window and
    the ordering all-reduce; else NCCL send/recv to itself. Growing n re-registers the window."""
    import torch

    import paper_1909_08006_b200 as ley

    ley.ley_set_option("dist_exchange_g1", exchange_g1)
    uid = ley.ley_comm_get_unique_id()
    comm = ley.ley_comm_init(1, 0, uid, 0)
    try:
        for n, dist in ((50_003, "skewed"), (20_000, "uniform"), (300_001, "three_keys")):
            recs = gen.records(n, seed=61, dist=dist)
            x = torch.from_numpy(recs).cuda()
            out = torch.empty_like(x)
            n_out, off = ley.ley_sort_dist(comm, x, n, out, n)
            torch.cuda.synchronize()
            assert (n_out, off) == (n, 0)
            assert np.array_equal(out.cpu().numpy(), oracle.sort(recs)[0])
            _, launches = ley.ley_stage_times()
            assert launches > 5  # the kernels this rank launched (the bench's gpu_launches at N > 1)
    finally:
        ley.ley_comm_destroy(comm)
        ley.ley_set_option("dist_exchange_g1", 0)


@pytest.mark.gpu
@pytest.mark.parametrize("stall_at", [1, 2, 4], ids=["first", "second", "fourth"])
def test_nccl_fault_times_out_and_aborts(cuda_ok, exchange_mode, stall_at):
    """NCCL fault handling ("any stage failure aborts the pipeline, reports the
    stage"). The dist_fault_stall hook holds the stream after the k-th collective of the call, as a peer
    that never completes it would. The library must not wait forever: within nccl_timeout_ms it aborts the
    communicator (ncclCommAbort), returns LEY_ERR_NCCL with the stage named in ley_last_error(), refuses
    further sorts on that communicator, lets ley_comm_destroy release it, and a new communicator works."""
    import time

    import torch

    import paper_1909_08006_b200 as ley

    n = 40_000
    recs = gen.records(n, seed=65, dist="uniform")
    x = torch.from_numpy(recs).cuda()
    out = torch.empty_like(x)
    ley.ley_set_option("dist_exchange_g1", 1)
    ley.ley_set_option("nccl_timeout_ms", 1500)
    comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
    try:
        ley.ley_set_option("dist_fault_stall", stall_at)
        t0 = time.monotonic()
        with pytest.raises(ley.LeyendaError) as ei:
            ley.ley_sort_dist(comm, x, n, out, n)
        took = time.monotonic() - t0
        assert ei.value.status == ley.LEY_ERR_NCCL
        msg = ley.ley_last_error()
        assert "communicator aborted" in msg and "dist" in msg, msg
        assert took < 1.5 + 10.0, took
        ley.ley_set_option("dist_fault_stall", 0)
        with pytest.raises(ley.LeyendaError) as ei:
            ley.ley_sort_dist(comm, x, n, out, n)
        assert ei.value.status == ley.LEY_ERR_NCCL and "aborted" in ley.ley_last_error()
    finally:
        ley.ley_set_option("dist_fault_stall", 0)
        ley.ley_comm_destroy(comm)
    torch.cuda.synchronize()
    comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
    try:
        assert ley.ley_sort_dist(comm, x, n, out, n) == (n, 0)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), oracle.sort(recs)[0])
    finally:
        ley.ley_comm_destroy(comm)
        ley.ley_set_option("dist_exchange_g1", 0)
        ley.ley_set_option("nccl_timeout_ms", 120000)


@pytest.mark.gpu
def test_nccl_pinned_host_slices(cuda_ok, exchange_mode):
    """ley_sort_dist with pinned host slices: staged on the device (H2D, the device path, D2H of the
    rank's range), with the exchange phases on; under a budget below slice + capacity (all ranks agree
    first) the external path runs instead and gives the same bytes."""
    import torch

    import paper_1909_08006_b200 as ley

    ley.ley_set_option("dist_exchange_g1", 1)
    comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
    try:
        n = 70_001
        recs = gen.records(n, seed=63, dist="skewed")
        x = torch.from_numpy(recs).pin_memory()
        out = torch.empty_like(x).pin_memory()
        n_out, off = ley.ley_sort_dist(comm, x, n, out, n)
        assert (n_out, off) == (n, 0)
        assert np.array_equal(out.numpy(), oracle.sort(recs)[0])
        # a budget below slice + capacity: the external path instead (same bytes)
        out.zero_()
        assert ley.ley_sort_dist(comm, x, n, out, n, device_budget_bytes=n * 100) == (n, 0)
        assert np.array_equal(out.numpy(), oracle.sort(recs)[0])
    finally:
        ley.ley_comm_destroy(comm)
        ley.ley_set_option("dist_exchange_g1", 0)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("dist", ["uniform", "skewed", "all_equal", "reverse"])
def test_external_loopback(cuda_ok, G, dist):
    """The multi-GPU EXTERNAL algorithm through the loopback: pinned host slices, a budget
    that forces many runs per rank, every rank's runs in one shared scratch, one partition, and each rank
    merging exactly floor((r+1)N/G) - floor(rN/G) records (boundary partitions merged by both neighbours,
    clipped); the concatenation is the oracle's output."""
    import torch

    import paper_1909_08006_b200 as ley

    N = 300_007
    recs = gen.records(N, seed=81 + G, dist=dist)
    rng = np.random.default_rng(G)
    cuts = np.sort(rng.integers(0, N, size=G - 1))
    n_local = np.diff(np.concatenate([[0], cuts, [N]])).tolist()
    if G > 2:
        n_local[0] += n_local[1]  # an empty rank
        n_local[1] = 0
    ins, outs, at = [], [], 0
    for r in range(G):
        ins.append(torch.from_numpy(recs[at * 100:(at + n_local[r]) * 100].copy()).pin_memory()
                   if n_local[r] else torch.empty(100, dtype=torch.uint8).pin_memory())
        at += n_local[r]
        outs.append(torch.empty((N // G + 2) * 100, dtype=torch.uint8).pin_memory())
    res = ley.ley_sort_dist_loopback(ins, n_local, outs, [N // G + 2] * G, device_budget_bytes=12 << 20)
    sizes, offs = _closed_form(N, G)
    assert [x[0] for x in res] == sizes and [x[1] for x in res] == offs
    got = np.concatenate([outs[r][: res[r][0] * 100].numpy() for r in range(G)])
    assert np.array_equal(got, oracle.sort(recs)[0])


@pytest.mark.gpu
def test_nccl_external_world_one(cuda_ok):
    """ley_sort_dist with pinned host slices whose staging exceeds the budget: the multi-GPU external path
    at world size 1 (runs, sample broadcast, partition, the rank's merge), equal to the oracle; a budget
    below its working set is refused (LEY_ERR_BUDGET) and the communicator stays usable."""
    import torch

    import paper_1909_08006_b200 as ley

    comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
    try:
        n = 400_001
        recs = gen.records(n, seed=85, dist="skewed")
        x = torch.from_numpy(recs).pin_memory()
        out = torch.empty_like(x).pin_memory()
        n_out, off = ley.ley_sort_dist(comm, x, n, out, n, device_budget_bytes=16 << 20)
        assert (n_out, off) == (n, 0)
        assert np.array_equal(out.numpy(), oracle.sort(recs)[0])
        with pytest.raises(ley.LeyendaError) as ei:
            ley.ley_sort_dist(comm, x, n, out, n, device_budget_bytes=1 << 20)
        assert ei.value.status == ley.LEY_ERR_BUDGET
        out.zero_()
        assert ley.ley_sort_dist(comm, x, n, out, n, device_budget_bytes=24 << 20) == (n, 0)
        assert np.array_equal(out.numpy(), oracle.sort(recs)[0])
    finally:
        ley.ley_comm_destroy(comm)


# ----------------------------------------------------------------------------------------- CPU (gloo)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, N, dist, q):
    import torch
    import torch.distributed as tdist

    import paper_1909_08006_b200 as ley

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        recs = gen.records(N, seed=77, dist=dist).reshape(N, 100)
        bounds = [0, N // 3, N] if world == 2 else [r * N // world for r in range(world + 1)]
        lo, hi = bounds[rank], bounds[rank + 1]
        local = recs[lo:hi]
        # K-s0 stand-in: local histogram of key bytes 0..1; C1: allreduce
        pref = local[:, 0].astype(np.int64) * 256 + local[:, 1]
        lh = np.bincount(pref, minlength=65536).astype(np.int64)
        gh = torch.from_numpy(lh.copy())
        tdist.all_reduce(gh)
        bins, rho, first = ley.ley_dist_plan_splitters(gh.numpy().astype(np.uint64), N, world)
        # K-s1 stand-in: boundary-bin candidates with global ordinals; C2: all-gather
        cand = [(bytes(local[i, :10]), lo + i) for i in range(hi - lo) if pref[i] in set(bins)]
        allc = [None] * world
        tdist.all_gather_object(allc, cand)
        cands = sorted(c for part in allc for c in part)
        spl = []
        for k in range(world - 1):
            start = sum(int(gh[b]) for b in sorted(set(bins)) if b < bins[k])
            spl.append(cands[start + rho[k]])
        # destinations; K-s2 + whole-bin counts must agree with a direct count
        dest = np.array([sum(1 for s in spl if s <= (bytes(local[i, :10]), lo + i)) for i in range(hi - lo)],
                        dtype=np.int64)
        direct = np.bincount(dest, minlength=world)
        whole = ley.ley_dist_bin_dest_counts(lh.astype(np.uint64), bins, world)
        extra = np.zeros(world, dtype=np.int64)
        for (kb, g) in cand:
            extra[sum(1 for s in spl if s <= (kb, g))] += 1
        assert np.array_equal(np.array(whole) + extra, direct)
        # C3: all-gather the send counts; exchange plan
        sc = torch.from_numpy(direct.copy())
        mat = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        tdist.all_gather(mat, sc)
        plan = ley.ley_dist_plan_exchange([m.tolist() for m in mat], world, rank)
        sizes, offs = _closed_form(N, world)
        assert plan["n_out"] == sizes[rank] and plan["out_offset"] == offs[rank]
        # K-p stand-in (stable partition) + C4 all-to-all-v
        order = np.argsort(dest, kind="stable")
        send = torch.from_numpy(np.ascontiguousarray(local[order]).reshape(-1))
        recv = torch.empty(plan["n_out"] * 100, dtype=torch.uint8)
        tdist.all_to_all_single(recv, send, [c * 100 for c in plan["recv_counts"]], [int(c) * 100 for c in direct])
        # the fused exchange's placement: every source writes its run for d at ley_dist_dest_offsets(...)[d]
        # of d's buffer; gathered here as (dest, offset, bytes), the pieces must tile each receive buffer
        # exactly and reproduce the all-to-all's result
        mlist = [m.tolist() for m in mat]
        doff = ley.ley_dist_dest_offsets(mlist, world, rank)
        seg = np.concatenate([[0], np.cumsum(direct)])
        pieces = [(d, doff[d], np.ascontiguousarray(local[order][seg[d]:seg[d + 1]]).tobytes()) for d in range(world)]
        allp = [None] * world
        tdist.all_gather_object(allp, pieces)
        placed = bytearray(plan["n_out"] * 100)
        cover = np.zeros(plan["n_out"], dtype=np.int64)
        for src_pieces in allp:
            for d, o, b in src_pieces:
                if d != rank:
                    continue
                placed[o * 100:o * 100 + len(b)] = b
                cover[o:o + len(b) // 100] += 1
        assert (cover == 1).all()
        assert bytes(placed) == recv.numpy().tobytes()
        for d in range(world):
            assert doff[d] == ley.ley_dist_plan_exchange(mlist, world, d)["recv_offsets"][rank]
        # local sort (oracle stands in for the GPU local sort); receive order = global order
        mine, _ = oracle.sort(recv.numpy())
        outs = [None] * world
        tdist.all_gather_object(outs, mine.tobytes())
        if rank == 0:
            got = b"".join(outs)
            q.put(got == oracle.sort(recs.reshape(-1))[0].tobytes())
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("dist", ["uniform", "skewed", "all_equal"])
def test_gloo_two_ranks_host_logic(dist):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, 3001, dist, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _shm_worker(rank, world, port, name, nbytes, q):
    import ctypes

    import torch.distributed as tdist

    import paper_1909_08006_b200 as ley

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        if rank == 0:
            addr = ley.ley_test_shared_scratch(name, nbytes, True)
            buf = (ctypes.c_uint8 * nbytes).from_address(addr)
            for i in range(0, nbytes, 4099):  # rank 0's "runs"
                buf[i] = (i * 7) & 0xFF
        tdist.barrier()
        if rank == 1:
            addr = ley.ley_test_shared_scratch(name, nbytes, False)
            buf = (ctypes.c_uint8 * nbytes).from_address(addr)
            ok = all(buf[i] == (i * 7) & 0xFF for i in range(0, nbytes, 4099))
            buf[1] = 0xAB  # written by rank 1, seen by rank 0
        tdist.barrier()
        if rank == 0:
            ok = buf[1] == 0xAB
        ley.ley_test_shared_scratch_close(addr, nbytes, name if rank == 0 else None)
        q.put((rank, ok))
    finally:
        tdist.destroy_process_group()


def test_gloo_shared_run_scratch():
    """The multi-GPU external path's shared host run scratch between two processes (host logic, CPU): rank 0
    creates and fills it, rank 1 opens the same name and sees the bytes, writes of either are seen by the
    other, and the name is removed afterwards."""
    import torch.multiprocessing as mp

    import paper_1909_08006_b200 as ley

    name, nbytes = f"/ley-test-{os.getpid()}", 1 << 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shm_worker, args=(r, 2, port, name, nbytes, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(q.get(timeout=10) for _ in range(2)) == [(0, True), (1, True)]
    with pytest.raises(ley.LeyendaError):  # unlinked: opening it again fails
        ley.ley_test_shared_scratch(name, nbytes, False)
