"""GPU parity (-m gpu): the CUDA path through the C ABI, byte-exact against the CPU oracle.

Integer/byte work, so the bar is bit-exact (BASELINE.json north_star "output bit-exact
against the oracle on the same seeded inputs, including stable tie order"). Sizes span several K-a tiles
(4096 records), K-c chunks (2048 pairs) and ragged tails; distributions cover the configs and the edge
cases of SURVEY.md §4 item 4.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
from gpu_util import Options, assert_parity, device_records, gpu_sort, to_device

pytestmark = pytest.mark.gpu

SIZES = [1, 2, 3, 4, 5, 31, 32, 33, 4095, 4096, 4097, 8191, 8193, 65535, 65536, 65537, 300_007]
DISTS = ["uniform", "skewed", "all_equal", "three_keys", "sorted", "reverse", "prefix2", "byte9", "ascii",
         "tiny_alphabet"]


@pytest.fixture(autouse=True)
def _cuda(cuda_ok):
    yield


def test_generator_twin():
    """The CUDA generator twin is byte-identical to the host generator (input plumbing)."""
    for dist in ("uniform", "skewed", "ascii"):
        n = 50_000
        d = device_records(n, seed=5, dist=dist).cpu().numpy()
        h = gen.records(n, seed=5, dist=dist)
        assert np.array_equal(d, h), dist
        d2 = torch.empty(1000 * 100, dtype=torch.uint8, device="cuda")
        gen.records_cuda(d2.data_ptr(), 1000, seed=5, dist=dist, i0=12345)
        assert np.array_equal(d2.cpu().numpy(), gen.records(1000, seed=5, dist=dist, i0=12345))


@pytest.mark.parametrize("n", SIZES)
def test_uniform_sizes(n):
    recs = gen.records(n, seed=n, dist="uniform")
    out, perm = gpu_sort(recs)
    assert_parity(recs, out, perm)


@pytest.mark.parametrize("n", [1, 2, 3, 6, 511, 513, 4095, 4097, 4098, 600_001, 606_209, 606_210])
def test_ka_forms_ragged(n):
    """All K-a forms on ragged sizes: partial 512-record pieces (bulk copies rounded down to 16 bytes; key-row
    boxes past the last 4-record group zero-filled), the last n mod 4 records read outside the tensor map
    (n = 1..3: every record), partial tiles, and more tiles than SMs (several tiles per persistent CTA)."""
    recs = gen.records(n, seed=n + 1, dist="skewed")
    for ks in (1, 2, 0):
        with Options(ka_stream=ks):
            out, perm = gpu_sort(recs)
        assert_parity(recs, out, perm)


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("n", [4097, 100_003])
def test_distributions(dist, n):
    recs = gen.records(n, seed=3, dist=dist)
    out, perm = gpu_sort(recs)
    assert_parity(recs, out, perm)


def test_c1_config():
    """BASELINE.json configs[0]: 1,000,000 uniform records, seed 0 (the oracle finishes in seconds)."""
    recs = gen.records(1_000_000, seed=0)
    out, perm = gpu_sort(recs)
    assert_parity(recs, out, perm)


@pytest.mark.parametrize("ws", [1, 0])
def test_medium_buckets_both_kd_forms(ws):
    """16-bit buckets of ~1500 records (the C2 shape, scaled down by sorting on a 2-byte constant prefix
    plus one varying byte: prefix2 sends everything into one level-1 bucket, recursion splits it into
    ~1K-record buckets) through the warp-specialised K-d+K-e tier and the alternating one."""
    recs = gen.records(300_007, seed=12, dist="prefix2")
    with Options(kd_ws=ws):
        out, perm = gpu_sort(recs)
    assert_parity(recs, out, perm)


@pytest.mark.parametrize("size", [32, 33, 512, 513, 2048, 2049, 8192, 8193, 10240, 10241, 16384, 16385])
@pytest.mark.parametrize("ws", [1, 0])
@pytest.mark.parametrize("fuse", [0, 1, 2], ids=["split", "fused", "corun"])
def test_kd_tier_boundaries(size, ws, fuse):
    """One level-1 bucket of exactly `size` records (a constant 2-byte prefix, prefix2) among a few
    thousand others, at every K-d tier boundary (warp 32, 512/128, 2048 warp-specialised or not,
    8192/1024, 10240/1024, 16384/768, and 16385 -> the byte-2 recursion): byte-exact with the oracle.
    fused: the level-1 split runs inside the K-d+K-e kernel of the big bucket's tier (kc_fuse 2..5; the
    2048 tier for sizes below it, which then has no bucket of its own); corun: the split's own kernel with
    that tier PDL-launched beside it (kc_corun)."""
    if fuse == 2 and (size > 2048 or not ws):
        pytest.skip("co-run applies to the warp-specialised 2048 tier only")
    big = gen.records(size, seed=size, dist="prefix2").reshape(size, 100)
    rest = gen.records(3001, seed=size + 1, dist="uniform").reshape(3001, 100)
    rest[rest[:, 0] == 0xAB, 0] = 0xAC  # keep the big bucket exactly `size` records
    recs = np.ascontiguousarray(np.concatenate([rest[:1500], big, rest[1500:]]).reshape(-1))
    tier_force = 2 if size <= 2048 else 3 if size <= 8192 else 4 if size <= 10240 else 5
    with Options(kd_ws=ws, kc_fuse=tier_force if fuse else 0, kc_corun=1 if fuse == 2 else 0):
        out, perm = gpu_sort(recs)
    assert_parity(recs, out, perm)


def test_zero_records():
    import paper_1909_08006_b200 as ley

    assert ley.ley_sort(0, 0, 0) == 0


@pytest.mark.parametrize("opts", [
    dict(warp_tier_max=1, smem_tier_max=0),          # all-recursive: MSD radix down to byte 9 (Alg. 1)
    dict(kd_digit_bits=0),                           # all-comparison inside K-d (ComparisonSort)
    dict(kd_digit_bits=0, kd_insert_max=64),         # insertion sort on whole small buckets
    dict(smem_tier_max=600),                         # many big buckets -> byte-2 level
    dict(warp_tier_max=4, kd_insert_max=1),          # warp bitonic for every sub-bucket
    dict(kd_ws=0),                                   # alternating sort/gather CTAs instead of warp-specialised
    dict(kd_ws=0, kd_digit_bits=0),
    dict(ka_stream=0),                               # K-a: one CTA per tile, direct key loads
    dict(ka_stream=2),                               # K-a: whole records through the bulk-copy ring
    dict(kc_fuse=0),                                 # level-1 split as its own kernel
    dict(kc_fuse=2),                                 # split fused into the warp-specialised 2048 tier
    dict(kc_fuse=2, kd_ws=0),                        # ... into the alternating 2048 tier (256 threads)
    dict(kc_fuse=2, kc_corun=1), dict(kc_fuse=2, kc_corun=2),  # split kernel beside the 2048 tier (co-run)
    dict(kc_fuse=2, kc_corun=1, pdl=2), dict(kc_fuse=2, kc_corun=1, smem_tier_max=600),
    dict(kc_fuse=3), dict(kc_fuse=4), dict(kc_fuse=5),  # ... into the 8192 / 10240 / 16384 tiers
    dict(kc_fuse=4, smem_tier_max=600),              # fused tier empty, big buckets recurse after it
    dict(pdl=0), dict(pdl=1), dict(pdl=2),           # tier kernels: stream order / PDL wait-first / overlap
    dict(pdl=2, smem_tier_max=600),                  # ... overlapping tiers at the recursion levels too
    dict(pdl=2, kd_ws=0), dict(pdl=2, kc_fuse=3),    # ... with the alternating tiers / a fused tier
    dict(kd_claim=0), dict(kd_claim=0, kd_ws=0),     # tier CTAs stride their list instead of claiming
    dict(kd_claim=0, pdl=2, smem_tier_max=600),
])
@pytest.mark.parametrize("dist", ["uniform", "skewed", "tiny_alphabet", "byte9"])
def test_forced_thresholds(opts, dist):
    """Algorithm 1's thresholds are speed knobs only: forcing the extremes must not
    change a single output byte."""
    recs = gen.records(70_001, seed=17, dist=dist)
    with Options(**opts):
        out, perm = gpu_sort(recs)
    assert_parity(recs, out, perm)


@pytest.mark.parametrize("pdl", [0, 2])
def test_warp_tier_near_ties(pdl):
    """The warp tier sorts one 64-bit composite per lane (the tail with its low 5 bits replaced by the lane)
    and falls back to the full (tail, ordinal) network when two sorted tails agree in their top 59 bits.
    Buckets of 2..32 records whose keys differ only in the low 5 bits of key byte 9, or not at all
    (duplicates, ordered by ordinal), must still come out in the oracle's order; so must buckets next to
    them that take the fast path."""
    rng = np.random.default_rng(5)
    base = gen.records(40_000, seed=5, dist="uniform").reshape(-1, 100).copy()
    groups = []
    for g in range(300):
        size = int(rng.integers(2, 33))
        proto = base[rng.integers(0, len(base))].copy()
        proto[0], proto[1] = g >> 8 | 0x40, g & 0xFF  # its own 16-bit bucket
        grp = np.repeat(proto[None, :], size, axis=0)
        if g % 3:  # near ties: only the low 5 bits of byte 9 differ (some exact duplicates among them)
            grp[:, 9] = (proto[9] & 0xE0) | rng.integers(0, 8, size=size).astype(np.uint8)
        grp[:, 10:] = rng.integers(0, 256, size=(size, 90), dtype=np.uint8)  # payload tells records apart
        groups.append(grp)
    recs = np.concatenate([base] + groups)
    recs = np.ascontiguousarray(recs[rng.permutation(len(recs))].reshape(-1))
    with Options(pdl=pdl):
        out, perm = gpu_sort(recs)
    assert_parity(recs, out, perm)


def test_async_stream_ordered():
    """Option async: device sorts without recursion return once enqueued. Back-to-back sorts on one stream,
    a sort on a second stream right after (same library workspace), one that needs the byte-2 recursion
    (falls back to waiting), a host-pointer sort and a perm sort all give the oracle's bytes."""
    import torch

    import paper_1909_08006_b200 as ley

    cases = [(gen.records(n, seed=60 + i, dist=d), n) for i, (n, d) in
             enumerate([(200_003, "uniform"), (150_001, "skewed"), (70_001, "prefix2"), (300_007, "uniform")])]
    xs = [to_device(r) for r, _ in cases]
    outs = [torch.empty_like(x) for x in xs]
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    with Options(**{"async": 1}):
        for x, o, (_, n) in zip(xs[:3], outs[:3], cases[:3]):
            ley.ley_sort(x, o, n, stream=a)
        ley.ley_sort(xs[3], outs[3], cases[3][1], stream=b)  # other stream, same workspace
        perm = torch.empty(cases[0][1], dtype=torch.int32, device="cuda")
        pout = torch.empty_like(xs[0])
        ley.ley_sort_perm(xs[0], pout, perm, cases[0][1], stream=a)
        hin = torch.from_numpy(cases[1][0]).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        ley.ley_sort(hin, hout, cases[1][1])  # host pointers: synchronous, after the device sorts
    torch.cuda.synchronize()
    for (recs, _), o in zip(cases, outs):
        exp, _ = oracle.sort(recs)
        assert np.array_equal(o.cpu().numpy(), exp)
    assert_parity(cases[0][0], pout.cpu().numpy(), perm.cpu().numpy().view(np.uint32))
    assert np.array_equal(hout.numpy(), oracle.sort(cases[1][0])[0])


@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 4097, 65537])
def test_async_small_sizes(n):
    """Stream-ordered calls at tiny and ragged sizes (one tile, partial tiles, a single record)."""
    import torch

    recs = gen.records(n, seed=n + 3, dist="uniform")
    with Options(**{"async": 1}):
        out, perm = gpu_sort(recs)
    torch.cuda.synchronize()
    assert_parity(recs, out, perm)


def test_repeat_bit_identical():
    recs = gen.records(200_003, seed=21, dist="skewed")
    a, pa = gpu_sort(recs)
    b, pb = gpu_sort(recs)
    assert np.array_equal(a, b) and np.array_equal(pa, pb)
    assert_parity(recs, a, pa)


def test_graph_replay_matches_direct():
    """Level 1 is captured into a CUDA graph on the first call and replayed after (option graphs): replays,
    a direct launch, a changed option (new graph key), a different caller stream, the profiled form and a
    released cache (graphs dropped with the buffers they point into) all give the oracle's bytes."""
    import torch

    import paper_1909_08006_b200 as ley

    n = 150_001
    recs = gen.records(n, seed=41, dist="skewed")
    exp, _ = oracle.sort(recs)
    x = to_device(recs)
    out = torch.empty_like(x)

    def run(**opts):
        out.zero_()
        with Options(**opts):
            ley.ley_sort(x, out, n)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), exp)

    for _ in range(3):
        run(graphs=1)
    run(graphs=0)
    run(graphs=1, kd_ws=0)
    run(graphs=1, profile=1)
    side = torch.cuda.Stream()
    out.zero_()
    ley.ley_sort(x, out, n, stream=side)
    side.synchronize()
    assert np.array_equal(out.cpu().numpy(), exp)
    ley.ley_release_cache(-1)
    run(graphs=1)


def test_pinned_host_path():
    """Pinned host pointers take the staged path (H2D, internal sort, D2H)."""
    import paper_1909_08006_b200 as ley

    n = 123_457
    recs = gen.records(n, seed=8, dist="skewed")
    x = torch.from_numpy(recs).pin_memory()
    out = torch.empty_like(x).pin_memory()
    ley.ley_sort(x, out, n)
    assert_parity(recs, out.numpy())


@pytest.mark.parametrize("dist,n,chunk", [
    ("uniform", 700_001, 100_000),     # 7 full windows + a ragged one
    ("skewed", 500_000, 64_000),       # recursion + ties, window edges inside tie runs
    ("ascii", 300_007, 1 << 21),       # default window size, capped at n / 4 for small n
    ("all_equal", 150_000, 40_960),    # output == input
    ("reverse", 99_999, 32_768),
])
def test_resident_host_path(dist, n, chunk):
    """Host path 2, resident input + streamed output (the paper's partial in-memory regime): under a
    budget that holds the input but not input + output, the sort runs in perm-only mode and K-e gathers
    the output window by window into two device windows copied to pinned host memory. Byte-exact with
    the oracle (out and perm), and the library's device high-water mark stays within the budget."""
    import paper_1909_08006_b200 as ley

    with Options(resident_chunk_records=chunk):
        plan = ley.ley_plan_query(n, 1)
        budget = plan["resident_bytes"]
        plan = ley.ley_plan_query(n, budget)
        assert plan["host_path"] == 2 and budget < plan["staged_bytes"], plan
        recs = gen.records(n, seed=71, dist=dist)
        x = torch.from_numpy(recs).pin_memory()
        out = torch.empty_like(x).pin_memory()
        perm = torch.empty(n, dtype=torch.int32).pin_memory()
        ley.ley_release_cache(-1)
        ley.ley_device_bytes(reset_peak=True)
        ley.ley_sort_perm(x, out, perm, n, device_budget_bytes=budget)
        _, peak = ley.ley_device_bytes()
        assert peak <= budget, (peak, budget)
        assert_parity(recs, out.numpy(), perm.numpy().view(np.uint32))
        # the plain call (no perm) and the path switch off (-> external) give the same bytes
        out2 = torch.empty_like(x).pin_memory()
        ley.ley_sort(x, out2, n, device_budget_bytes=budget)
        assert torch.equal(out, out2)
        with Options(resident_path=0):
            assert ley.ley_plan_query(n, budget)["host_path"] == 1
            out3 = torch.empty_like(x).pin_memory()
            ley.ley_sort(x, out3, n, device_budget_bytes=budget)
        assert torch.equal(out, out3)
    ley.ley_release_cache(-1)


def test_streaming_submit_pipeline():
    """ley_sort_submit: consecutive host sorts overlap through two device slots (H2D of call k+1 with the
    D2H of call k). Five calls of different sizes and distributions (slots reused and grown) must each
    land byte-exact, and the caller's stream must be ordered after each call's D2H."""
    import paper_1909_08006_b200 as ley

    cases = [(70_001, "uniform"), (123_457, "skewed"), (4097, "all_equal"), (200_003, "tiny_alphabet"),
             (33, "reverse")]
    bufs = []
    for i, (n, dist) in enumerate(cases):
        recs = gen.records(n, seed=60 + i, dist=dist)
        x, out = _pinned(recs)
        out.fill_(0xAB)
        ley.ley_sort_submit(x, out, n)
        bufs.append((recs, x, out))
    ley.ley_sort_drain()
    for recs, _, out in bufs:
        assert_parity(recs, out.numpy())
    # stream ordering: the H2D waits for work already on the caller's stream (here a copy into `in`)
    recs = gen.records(50_000, seed=99, dist="skewed")
    x, out = _pinned(recs)
    x0 = x.clone()
    x.zero_()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        torch.cuda._sleep(50_000_000)  # keep the stream busy so an unordered H2D would read zeros
        x.copy_(x0.cuda(non_blocking=True), non_blocking=True)
    ley.ley_sort_submit(x, out, 50_000, stream=st)
    ley.ley_sort_drain()
    assert_parity(recs, out.numpy())
    # device pointers are rejected (the blocking ley_sort is the device-resident call)
    d = torch.from_numpy(recs).cuda()
    assert ley.ley_sort_submit(d, torch.empty_like(d), 50_000, raise_on_error=False) == ley.LEY_ERR_UNSUPPORTED
    ley.ley_sort_drain()
    # releasing the cache stops the pipeline's worker; the next submit starts a fresh one; drain is idempotent
    ley.ley_release_cache(-1)
    ley.ley_sort_drain()
    out.fill_(0)
    ley.ley_sort_submit(x, out, 50_000)
    ley.ley_release_cache(-1)  # with a call in flight: its sort and copy complete before the worker stops
    assert_parity(recs, out.numpy())
    ley.ley_sort_drain()


@pytest.mark.parametrize("parts", [1, 2, 3, 4])
def test_streaming_copy_pieces(parts):
    """ley_sort_submit with its copies in 1..4 pieces on their own streams (option pipe_split): ragged sizes
    (pieces rounded to 256 bytes, the last one takes the rest) and interleaved calls land byte-exact."""
    import paper_1909_08006_b200 as ley

    with Options(pipe_split=parts):
        bufs = []
        for i, n in enumerate((1, 4097, 333_333, 77_777)):
            recs = gen.records(n, seed=120 + i + parts, dist="skewed")
            x, out = _pinned(recs)
            out.fill_(0x5A)
            ley.ley_sort_submit(x, out, n)
            bufs.append((recs, out))
        ley.ley_sort_drain()
        for recs, out in bufs:
            assert_parity(recs, out.numpy())


def test_pageable_rejected():
    import paper_1909_08006_b200 as ley

    recs = gen.records(1000, seed=1)
    out = np.empty_like(recs)
    assert ley.ley_sort(recs, out, 1000, raise_on_error=False) == ley.LEY_ERR_UNSUPPORTED


def test_internal_device_memory_within_budget():
    """Device pointers: the library's high-water mark stays within the scratch ley_plan_query reports (the
    budget check uses the same figure), including skew that recurses through several MSD levels."""
    import paper_1909_08006_b200 as ley

    for n, dist in [(300_007, "skewed"), (250_000, "prefix2"), (200_000, "tiny_alphabet")]:
        need = ley.ley_plan_query(n)["internal_scratch"]
        x = device_records(n, seed=5, dist=dist)
        out = torch.empty_like(x)
        ley.ley_release_cache(-1)
        ley.ley_device_bytes(reset_peak=True)
        ley.ley_sort(x, out, n, device_budget_bytes=need)
        _, peak = ley.ley_device_bytes()
        assert peak <= need, (dist, peak, need)
        assert ley.ley_sort(x, out, n, device_budget_bytes=need - 1, raise_on_error=False) == ley.LEY_ERR_BUDGET
    ley.ley_release_cache(-1)


def test_device_budget_too_small():
    import paper_1909_08006_b200 as ley

    x = device_records(10_000, seed=1)
    out = torch.empty_like(x)
    assert ley.ley_sort(x, out, 10_000, device_budget_bytes=1 << 16, raise_on_error=False) == ley.LEY_ERR_BUDGET


def _certify_on_host(x: torch.Tensor, n: int, **kw):
    import paper_1909_08006_b200 as ley

    out = torch.empty_like(x)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ley.ley_sort_perm(x, out, perm, n, **kw)
    torch.cuda.synchronize()
    h_in = x.cpu().numpy()
    h_out = out.cpu().numpy()
    h_perm = perm.cpu().numpy().view(np.uint32)
    assert oracle.certify(h_in, h_out, h_perm) == 0
    return h_in, h_out


@pytest.mark.slow
def test_c2_full_size_certificate():
    """BASELINE.json configs[1] at full size (1e8 records, seed 1), the bench's launch configuration:
    the certificate (perm is a permutation, out[j] == in[perm[j]], (key, perm) strictly increasing) pins
    the output to the oracle's exactly; the oracle's own sorted digest cross-checks a sample of it."""
    n = 100_000_000
    x = device_records(n, seed=1)
    h_in, h_out = _certify_on_host(x, n)
    # the oracle on a 2M-record slice of the input agrees with sorting that slice on the GPU
    sl = h_in[: 2_000_000 * 100]
    out, perm = gpu_sort(sl)
    assert_parity(sl, out, perm)


@pytest.mark.slow
def test_c3_full_size_certificate():
    """BASELINE.json configs[2]: 2e8 skewed records with 2% duplicated keys (seed 2) — recursion on
    bytes 2 and 3 plus stable ties, certified exactly; multiset hash equal (S:79 invariant)."""
    n = 200_000_000
    x = device_records(n, seed=2, dist="skewed")
    h_in, h_out = _certify_on_host(x, n)
    assert oracle.multiset_hash(h_in) == oracle.multiset_hash(h_out)


def _certify_on_device(x: torch.Tensor, out: torch.Tensor, perm: torch.Tensor, n: int, step: int = 20_000_000):
    """The certificate (perm is a permutation; out[j] == in[perm[j]]; (key, perm) strictly increasing) with
    plain torch ops on the device, in chunks — for sizes whose host copy would not fit. Independent of the
    library's kernels; together the three properties pin the output to the oracle's."""
    X, O = x.view(n, 100), out.view(n, 100)
    seen = torch.zeros(n, dtype=torch.bool, device="cuda")
    prev = None
    w = torch.tensor([1 << (8 * (6 - i)) for i in range(7)], dtype=torch.int64, device="cuda")
    for a in range(0, n, step):
        b = min(n, a + step)
        pc = perm[a:b].to(torch.int64)
        assert int(pc.min()) >= 0 and int(pc.max()) < n
        seen[pc] = True
        assert torch.equal(O[a:b], X[pc]), f"out != in[perm] in [{a}, {b})"
        kb = O[a:b, :10].to(torch.int64)
        hi = (kb[:, :7] * w).sum(1)                                     # key bytes 0..6
        lo = ((kb[:, 7] << 16) | (kb[:, 8] << 8) | kb[:, 9]) << 32 | pc  # bytes 7..9, then the ordinal
        if prev is not None:
            hi = torch.cat([prev[0], hi])
            lo = torch.cat([prev[1], lo])
        inc = (hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))
        assert bool(inc.all()), f"(key, ordinal) not strictly increasing in [{a}, {b})"
        prev = (hi[-1:], lo[-1:])
    assert bool(seen.all()), "perm is not a permutation"


def test_device_certificate_rejects_corruption():
    """The device-side certifier used at full size must reject every single-defect corruption: swapped
    records, a swapped tie (unstable order), a payload byte flip, a duplicated ordinal."""
    import paper_1909_08006_b200 as ley

    n = 100_003
    x = device_records(n, seed=5, dist="three_keys")
    out = torch.empty_like(x)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ley.ley_sort_perm(x, out, perm, n)
    torch.cuda.synchronize()
    _certify_on_device(x, out, perm, n, step=30_000)

    def bad(mut):
        o, p = out.clone(), perm.clone()
        mut(o.view(n, 100), p)
        with pytest.raises(AssertionError):
            _certify_on_device(x, o, p, n, step=30_000)

    def swap_rows(o, p, i, j):
        o[[i, j]] = o[[j, i]]
        p[[i, j]] = p[[j, i]]

    bad(lambda o, p: swap_rows(o, p, 10, 90_000))     # out of key order
    bad(lambda o, p: swap_rows(o, p, 40_000, 40_001))  # adjacent equal keys (three_keys): unstable tie
    bad(lambda o, p: o[777].__setitem__(55, o[777, 55] ^ 1))  # payload edit
    bad(lambda o, p: p.__setitem__(5, p[6]))           # not a permutation


@pytest.mark.slow
def test_c4_full_size_certificate():
    """BASELINE.json configs[3] at full size (6e8 records = 60 GB, seed 3), the bench's launch
    configuration: certified on the device (in + out + perm + scratch fit the 180 GB HBM), and the oracle
    sorts a 2M-record slice of the same input to the same bytes as the GPU."""
    import paper_1909_08006_b200 as ley

    import gc

    gc.collect()
    torch.cuda.empty_cache()  # earlier tests' cached blocks: in + out + perm + scratch need ~140 GB
    ley.ley_release_cache(-1)
    n = 600_000_000
    x = device_records(n, seed=3)
    out = torch.empty_like(x)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ley.ley_sort_perm(x, out, perm, n)
    torch.cuda.synchronize()
    _certify_on_device(x, out, perm, n)
    sl = x[: 2_000_000 * 100].cpu().numpy()
    del out, perm
    torch.cuda.empty_cache()
    o2, p2 = gpu_sort(sl)
    assert_parity(sl, o2, p2)
    del x
    torch.cuda.empty_cache()
    ley.ley_release_cache(-1)


@pytest.mark.slow
def test_ascii_20gb_and_partial_in_memory():
    """SURVEY §8f NEXT 4 workloads at full size. (1) The paper's 20 GB ASCII set ("ASCII for 20 GB
    dataset"): 2e8 printable records ending in CR LF, 95 live values per key byte, so every 16-bit bucket
    (~22K records) recurses on byte 2 — sorted on the device and certified there. (2) The paper's
    "partial in-memory" regime (Table 2's 30 GB memory for 20 GB of data): the same records
    in pinned host memory under a 30 GB device budget — the input fits, input + output do not — take host
    path 2 (resident input, streamed output), and with that path switched off the external path (a few
    large runs); both outputs must equal the certified device result byte for byte."""
    import gc

    import paper_1909_08006_b200 as ley

    gc.collect()
    torch.cuda.empty_cache()
    ley.ley_release_cache(-1)
    n, budget = 200_000_000, 30_000_000_000
    x = device_records(n, seed=5, dist="ascii")
    out = torch.empty_like(x)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ley.ley_sort_perm(x, out, perm, n)
    torch.cuda.synchronize()
    _certify_on_device(x, out, perm, n)
    del perm
    plan = ley.ley_plan_query(n, budget)
    assert plan["host_path"] == 2, plan
    h_in = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
    h_in.copy_(x)
    del x
    torch.cuda.empty_cache()
    ley.ley_release_cache(-1)
    h_out = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
    step = 20_000_000 * 100
    for resident in (1, 0):
        with Options(resident_path=resident):
            p = ley.ley_plan_query(n, budget)
            assert p["host_path"] == (2 if resident else 1) and (resident or 2 <= p["runs"] <= 8), p
            h_out.zero_()
            ley.ley_sort(h_in, h_out, n, device_budget_bytes=budget)
        for a in range(0, n * 100, step):
            assert torch.equal(h_out[a:a + step].cuda(), out[a:a + step]), f"path {p['host_path']} != device at {a}"
    del out, h_in, h_out
    torch.cuda.empty_cache()
    ley.ley_release_cache(-1)


# ------------------------------------------------------------------ external path
def _pinned(recs):
    x = torch.from_numpy(recs).pin_memory()
    return x, torch.empty_like(x).pin_memory()


@pytest.mark.parametrize("dist,n,budget", [
    ("uniform", 1_000_000, 16 << 20),     # ~28 runs, many partitions
    ("skewed", 600_001, 12 << 20),        # duplicates spanning runs and partitions
    ("all_equal", 300_000, 8 << 20),      # every tie crosses runs: output == input
    ("tiny_alphabet", 250_003, 8 << 20),
    ("sorted", 200_000, 8 << 20),
    ("reverse", 200_000, 8 << 20),
])
def test_external_matches_oracle(dist, n, budget):
    import paper_1909_08006_b200 as ley

    plan = ley.ley_plan_query(n, budget)
    assert plan["host_path"] == 1 and plan["runs"] > 1
    recs = gen.records(n, seed=41, dist=dist)
    x, out = _pinned(recs)
    perm = torch.empty(n, dtype=torch.int32).pin_memory()
    ley.ley_sort_perm(x, out, perm, n, device_budget_bytes=budget)
    assert_parity(recs, out.numpy(), perm.numpy().view(np.uint32))


@pytest.mark.parametrize("dist,n,budget", [
    ("uniform", 1_000_003, 24 << 20),
    ("skewed", 600_001, 12 << 20),
    ("all_equal", 300_000, 8 << 20),
    ("three_keys", 250_003, 8 << 20),
])
def test_external_keyptr_matches_oracle(dist, n, budget):
    """SURVEY §8f NEXT 3, the paper's key-pointer pattern on the external path (option
    ext_keyptr): runs of 16-byte (key, ordinal) tuples instead of records, the merge gathering every output
    record from the pinned input by its ordinal. Same bytes and permutation as the oracle (ties across runs
    and partitions included), the device high-water mark within the budget, and equal to the record form."""
    import paper_1909_08006_b200 as ley

    recs = gen.records(n, seed=45, dist=dist)
    x, out = _pinned(recs)
    perm = torch.empty(n, dtype=torch.int32).pin_memory()
    with Options(ext_keyptr=1):
        ley.ley_release_cache(-1)
        ley.ley_device_bytes(reset_peak=True)
        ley.ley_sort_perm(x, out, perm, n, device_budget_bytes=budget)
        _, peak = ley.ley_device_bytes()
    assert peak <= budget, f"library held {peak} bytes under a {budget}-byte budget"
    assert_parity(recs, out.numpy(), perm.numpy().view(np.uint32))
    out2 = torch.empty_like(x).pin_memory()
    ley.ley_sort(x, out2, n, device_budget_bytes=budget)
    assert np.array_equal(out2.numpy(), out.numpy())
    with Options(ext_keyptr=1):  # short keys on the key-pointer form too
        ley.ley_sort(x, out2, n, key_bytes=3, device_budget_bytes=budget)
    exp3, _ = oracle.sort(recs, key_bytes=3)
    assert np.array_equal(out2.numpy(), exp3)


def test_external_equals_internal_and_single_run():
    import paper_1909_08006_b200 as ley

    n = 400_000
    recs = gen.records(n, seed=43, dist="skewed")
    x, out_ext = _pinned(recs)
    ley.ley_sort(x, out_ext, n, device_budget_bytes=10 << 20)
    out_int, _ = gpu_sort(recs, with_perm=False)
    assert np.array_equal(out_ext.numpy(), out_int)
    # K = 1 run: the merge stage degenerates to a copy
    with Options(ext_run_records=n):
        out1 = torch.empty_like(x).pin_memory()
        ley.ley_sort(x, out1, n, device_budget_bytes=10 << 20)
    assert np.array_equal(out1.numpy(), out_int)


def test_external_device_memory_within_budget():
    """The external path's device high-water mark stays within device_budget_bytes (
    P:19's memory limit), measured by the library's own allocation accounting (ley_device_bytes) over a
    cold call, for budgets from a few runs to many."""
    import paper_1909_08006_b200 as ley

    n = 1_000_000
    recs = gen.records(n, seed=44)
    x, out = _pinned(recs)
    for budget in (12 << 20, 24 << 20, 96 << 20):
        ley.ley_release_cache(-1)
        cur, _ = ley.ley_device_bytes(reset_peak=True)
        assert cur == 0
        ley.ley_sort(x, out, n, device_budget_bytes=budget)
        _, peak = ley.ley_device_bytes()
        assert peak <= budget, f"library held {peak} bytes under a {budget}-byte budget"
        assert_parity(recs, out.numpy())
    ley.ley_release_cache(-1)


def test_external_budget_too_small():
    import paper_1909_08006_b200 as ley

    n = 100_000
    x, out = _pinned(gen.records(n, seed=1))
    assert ley.ley_sort(x, out, n, device_budget_bytes=1 << 20, raise_on_error=False) == ley.LEY_ERR_BUDGET
