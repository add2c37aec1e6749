"""Flexible key sizes (§5 P:164 "flexible key sizes ... a prefix generator for all types of keys";
SURVEY.md §8f NEXT 4): key = record bytes [0, key_bytes), 1..100, stable by input index.

Keys of <= 10 bytes run one pass whose sort key carries the ordinal in its unused bytes; longer keys run
LSD passes over the 10-byte windows. Every result is compared byte for byte (records and permutation) with
the oracle's record-comparison sort (oracle.sort(..., key_bytes=k), pinned in tests/test_oracle.py).
"""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu


def _records(n, seed, dist):
    """Generator records with low-entropy bytes 10..39 (copies of key bytes mod 3), so keys longer than
    10 bytes keep long tie runs for their later windows to break."""
    r = gen.records(n, seed=seed, dist=dist).reshape(n, 100)
    r[:, 10:40] = r[:, 0:30] % 3
    return np.ascontiguousarray(r.reshape(-1))


def _expect(recs, k):
    return oracle.sort(recs, key_bytes=k)


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 9, 10, 11, 15, 20, 37, 100])
@pytest.mark.parametrize("dist", ["uniform", "tiny_alphabet", "three_keys"])
def test_device_path(cuda_ok, k, dist):
    import paper_1909_08006_b200 as ley

    n = 150_003
    recs = _records(n, 90 + k, dist)
    x = torch.from_numpy(recs).cuda()
    out = torch.empty_like(x)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ley.ley_sort_perm(x, out, perm, n, key_bytes=k)
    exp, eperm = _expect(recs, k)
    assert np.array_equal(out.cpu().numpy(), exp)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), eperm)
    out2 = torch.empty_like(x)
    ley.ley_sort(x, out2, n, key_bytes=k)  # no perm: the multi-pass path without compositions
    assert torch.equal(out, out2)


@pytest.mark.parametrize("groups", [0, 40, 3000, 100, 1])
@pytest.mark.parametrize("hybrid", [1, 0])
def test_long_keys_tie_groups(cuda_ok, groups, hybrid):
    """Keys of 24 bytes whose 10-byte prefixes tie in controlled ways: none (uniform), 40 large groups of
    ~5000 (window passes on each slice), 3000 groups of ~67 (a CTA per group), 100 groups of ~2000 (more
    large groups than the hybrid handles: the plain window passes), one group holding every record; plus
    small groups of 2..32 around them. The hybrid (key_hybrid=1) and the plain LSD passes (0) must both
    equal the oracle."""
    import paper_1909_08006_b200 as ley

    n = 200_001
    r = gen.records(n, seed=33 + groups, dist="uniform").reshape(n, 100)
    rng = np.random.default_rng(groups)
    if groups:  # prefix = group id (big-endian in bytes 6..9), bytes 0..5 zero
        g = rng.integers(0, groups, size=n).astype(np.uint32)
        r[:, :10] = 0
        for b in range(4):
            r[:, 9 - b] = (g >> (8 * b)) & 0xFF
    # small groups: every 10th record joins a pair (or a few) sharing a fresh prefix 0xFF ++ (i // 20)
    idx = np.arange(0, n, 10)
    pid = (idx // 20).astype(np.uint64)
    r[idx, 0], r[idx, 1] = 0xFF, 0
    for b in range(8):
        r[idx, 9 - b] = (pid >> np.uint64(8 * b)) & np.uint64(0xFF)
    r[:, 10:24] = rng.integers(0, 3, size=(n, 14))  # the rest of the key: low entropy -> deep ties
    recs = np.ascontiguousarray(r.reshape(-1))
    x = torch.from_numpy(recs).cuda()
    out = torch.empty_like(x)
    ley.ley_set_option("key_hybrid", hybrid)
    try:
        ley.ley_sort(x, out, n, key_bytes=24)
    finally:
        ley.ley_set_option("key_hybrid", 1)
    assert np.array_equal(out.cpu().numpy(), _expect(recs, 24)[0])


def _grouped(n, sizes, seed):
    """n records whose 10-byte prefixes come in runs of the given sizes (cycled; distinct prefixes, shuffled
    positions), key bytes 10..23 low-entropy."""
    rng = np.random.default_rng(seed)
    r = gen.records(n, seed=seed, dist="uniform").reshape(n, 100)
    gid = np.repeat(np.arange(n, dtype=np.uint64), np.resize(np.asarray(sizes), n))[:n]
    gid = gid[rng.permutation(n)] * np.uint64(2654435761) + np.uint64(12345)  # distinct, scattered prefixes
    r[:, 0:2] = 7
    for b in range(8):
        r[:, 9 - b] = (gid >> np.uint64(8 * b)) & np.uint64(0xFF)
    r[:, 10:24] = rng.integers(0, 3, size=(n, 14))
    return np.ascontiguousarray(r.reshape(-1))


@pytest.mark.parametrize("sizes", [[32, 33], [31, 32, 33, 34, 2], [2, 3, 5], [7, 8, 9, 1], [64, 1, 1],
                                   [1024, 1025], [500, 67, 2]])
def test_tie_group_sizes(cuda_ok, sizes):
    """Groups at the eight-lane boundary (7 tiny, 8 and 9 to the warp pass), the warp boundary (32 warp,
    33 CTA), the CTA boundary (1024 CTA, 1025 large) and many tiny groups (about 10^5), all found and fixed
    on the device; the few large ones go through the window passes on their slices."""
    import paper_1909_08006_b200 as ley

    n = 300_000 if max(sizes) <= 9 else 30 * sum(sizes)  # <= 64 large groups when they exist
    recs = _grouped(n, sizes, 5 + len(sizes))
    x = torch.from_numpy(recs).cuda()
    out = torch.empty_like(x)
    ley.ley_sort(x, out, n, key_bytes=24)
    assert np.array_equal(out.cpu().numpy(), _expect(recs, 24)[0])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tie_scan_digest_collision(cuda_ok, seed):
    """The tie-group scan reads the prefix digests K-e writes (k_bucket.cu prefix_digest) and verifies
    equal-digest neighbours on the records. Two different 10-byte prefixes A, B built to share a digest,
    adjacent in sorted order (fillers sort before/after them), 12 records each: treating them as one tie
    group of 24 would reorder A's and B's records together by bytes 10.. — the result must equal the oracle."""
    import paper_1909_08006_b200 as ley

    C = 0x9E3779B97F4A7C15  # white-box: the digest's multiplier (words 0-1 XOR (bytes 8-9) * C, mod 2^64)
    rng = np.random.default_rng(seed)
    while True:
        x = int(rng.integers(0, 2**63)) | (int(rng.integers(0, 2)) << 63)
        a, b = (int(v) for v in rng.integers(0, 1 << 16, size=2))
        y = x ^ ((a * C) & (2**64 - 1)) ^ ((b * C) & (2**64 - 1))
        if a != b and all(0 < (v & 0xFF) < 0xFF for v in (x, y)):
            break
    n = 100_000
    r = gen.records(n, seed=70 + seed, dist="uniform").reshape(n, 100)
    r[: n // 2, 0], r[n // 2:, 0] = 0x00, 0xFF
    at = rng.permutation(n)[:24]
    for j, pos in enumerate(at):
        lo, hi = (x, a) if j < 12 else (y, b)
        r[pos, 0:8] = np.frombuffer(lo.to_bytes(8, "little"), dtype=np.uint8)
        r[pos, 8:10] = np.frombuffer(hi.to_bytes(2, "little"), dtype=np.uint8)
    r[:, 10:20] = rng.integers(0, 3, size=(n, 10))
    recs = np.ascontiguousarray(r.reshape(-1))
    x_t = torch.from_numpy(recs).cuda()
    out = torch.empty_like(x_t)
    ley.ley_sort(x_t, out, n, key_bytes=20)
    assert np.array_equal(out.cpu().numpy(), _expect(recs, 20)[0])


@pytest.mark.parametrize("k", [1, 4, 12])
def test_large_and_skewed(cuda_ok, k):
    """Skewed C3-style keys at 2M records (recursion below the key prefix) with short and long keys."""
    import paper_1909_08006_b200 as ley

    n = 2_000_000
    recs = _records(n, 7, "skewed")
    x = torch.from_numpy(recs).cuda()
    out = torch.empty_like(x)
    ley.ley_sort(x, out, n, key_bytes=k)
    assert np.array_equal(out.cpu().numpy(), _expect(recs, k)[0])


def test_host_paths(cuda_ok):
    """Staged (k = 20), resident (k = 4), external (k = 3 and 9) and streaming (k = 15) host paths; the
    external and resident paths refuse keys longer than 10 bytes."""
    import paper_1909_08006_b200 as ley

    n = 400_001
    recs = _records(n, 5, "tiny_alphabet")
    x = torch.from_numpy(recs).pin_memory()

    def run(k, budget=0):
        out = torch.empty_like(x).pin_memory()
        perm = torch.empty(n, dtype=torch.int32).pin_memory()
        ley.ley_sort_perm(x, out, perm, n, key_bytes=k, device_budget_bytes=budget)
        exp, eperm = _expect(recs, k)
        assert np.array_equal(out.numpy(), exp), k
        assert np.array_equal(perm.numpy().view(np.uint32), eperm), k

    run(20)                                                  # staged
    res_budget = ley.ley_plan_query(n, 1)["resident_bytes"]
    assert ley.ley_plan_query(n, res_budget)["host_path"] == 2
    run(4, res_budget)                                       # resident
    for k in (3, 9):
        run(k, 12 << 20)                                     # external, several runs
    out = torch.empty_like(x).pin_memory()
    assert ley.ley_sort(x, out, n, key_bytes=11, device_budget_bytes=12 << 20,
                        raise_on_error=False) == ley.LEY_ERR_UNSUPPORTED
    # streaming submit
    outs = [torch.empty_like(x).pin_memory() for _ in range(2)]
    for o in outs:
        ley.ley_sort_submit(x, o, n, key_bytes=15)
    ley.ley_sort_drain()
    exp = _expect(recs, 15)[0]
    for o in outs:
        assert np.array_equal(o.numpy(), exp)


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("k", [1, 2, 5])
def test_dist_loopback(cuda_ok, fused, k):
    """The multi-GPU algorithm (loopback, G = 4, one empty rank) with short keys: splitters, destinations
    and the local sorts all compare the k-byte prefix, ties by global ordinal."""
    import paper_1909_08006_b200 as ley

    ley.ley_set_option("dist_fused", fused)
    try:
        G, N = 4, 80_001
        recs = _records(N, 11 + k, "tiny_alphabet")
        n_local = [30_000, 0, 25_000, N - 55_000]
        ins, outs, at = [], [], 0
        for r in range(G):
            part = recs[at * 100:(at + n_local[r]) * 100]
            at += n_local[r]
            ins.append(torch.from_numpy(part.copy()).cuda() if n_local[r] else torch.empty(100, dtype=torch.uint8,
                                                                                           device="cuda"))
            outs.append(torch.empty((N // G + 2) * 100, dtype=torch.uint8, device="cuda"))
        res = ley.ley_sort_dist_loopback(ins, n_local, outs, [N // G + 2] * G, key_bytes=k)
        assert [x[0] for x in res] == [((r + 1) * N // G) - (r * N // G) for r in range(G)]
        got = np.concatenate([outs[r][: res[r][0] * 100].cpu().numpy() for r in range(G)])
        assert np.array_equal(got, _expect(recs, k)[0])
    finally:
        ley.ley_set_option("dist_fused", 1)


@pytest.mark.parametrize("k", [2, 7])
def test_dist_external_loopback(cuda_ok, k):
    """The multi-GPU external algorithm (loopback, G = 3, pinned host slices, many runs) with short keys:
    merge composites and slice searches compare the k-byte prefix, ties by global input order."""
    import paper_1909_08006_b200 as ley

    G, N = 3, 150_001
    recs = _records(N, 30 + k, "tiny_alphabet")
    n_local = [60_000, 40_000, N - 100_000]
    ins, outs, at = [], [], 0
    for r in range(G):
        ins.append(torch.from_numpy(recs[at * 100:(at + n_local[r]) * 100].copy()).pin_memory())
        at += n_local[r]
        outs.append(torch.empty((N // G + 2) * 100, dtype=torch.uint8).pin_memory())
    res = ley.ley_sort_dist_loopback(ins, n_local, outs, [N // G + 2] * G, key_bytes=k, device_budget_bytes=12 << 20)
    got = np.concatenate([outs[r][: res[r][0] * 100].numpy() for r in range(G)])
    assert np.array_equal(got, _expect(recs, k)[0])


def test_nccl_world_one_exchange(cuda_ok):
    import paper_1909_08006_b200 as ley

    ley.ley_set_option("dist_exchange_g1", 1)
    comm = ley.ley_comm_init(1, 0, ley.ley_comm_get_unique_id(), 0)
    try:
        n = 60_007
        recs = _records(n, 3, "three_keys")
        x = torch.from_numpy(recs).cuda()
        out = torch.empty_like(x)
        n_out, off = ley.ley_sort_dist(comm, x, n, out, n, key_bytes=3)
        assert (n_out, off) == (n, 0)
        assert np.array_equal(out.cpu().numpy(), _expect(recs, 3)[0])
        with pytest.raises(ley.LeyendaError) as ei:
            ley.ley_sort_dist(comm, x, n, out, n, key_bytes=11)
        assert ei.value.status == ley.LEY_ERR_UNSUPPORTED
    finally:
        ley.ley_comm_destroy(comm)
        ley.ley_set_option("dist_exchange_g1", 0)


def test_invalid_key_bytes(cuda_ok):
    import paper_1909_08006_b200 as ley

    x = torch.zeros(100 * 10, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(x)
    for k in (0, 101):
        assert ley.ley_sort(x, out, 10, key_bytes=k, raise_on_error=False) == ley.LEY_ERR_UNSUPPORTED
