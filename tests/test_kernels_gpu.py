"""Kernel unit tests (-m gpu): single kernels of the path through the C-ABI
verification hooks, each against a plain CPU model written here from its definition.

* K-b (`ley_test_scan_excl`): the decoupled-look-back exclusive scan == a sequential prefix sum
  (numpy cumsum), for lengths that give 1, 2, 3, ... look-back tiles and a ragged tail.
* K-a (`ley_test_tile_sort`, both forms): per 4096-record tile, the byte-0 counts == a naive tally, the
  tile-local offsets == their exclusive prefix, hist16 == a tally of 2-byte prefixes, and every tile's
  pairs are the tile's (key bytes 1..9, local index) in byte-0 order (as a multiset per byte-0 run).
"""
import numpy as np
import pytest
import torch

import gen
import paper_1909_08006_b200 as ley

pytestmark = pytest.mark.gpu
TILE = 4096


@pytest.fixture(autouse=True)
def _cuda(cuda_ok):
    yield


@pytest.mark.parametrize("m", [1, 2, 4095, 4096, 4097, 3 * 4096 + 5, 1000 * 4096 + 17, 100_003, 2_500_001])
def test_kb_scan_matches_prefix_sum(m):
    rng = np.random.default_rng(m)
    a = rng.integers(0, 1000, size=m, dtype=np.uint32)
    d_in = torch.from_numpy(a.view(np.int32)).cuda()
    d_out = torch.full((m + 1,), -1, dtype=torch.int32, device="cuda")
    ley.ley_test_scan_excl(d_in, d_out, m)
    out = d_out.cpu().numpy().view(np.uint32)
    exp = np.concatenate([[0], np.cumsum(a, dtype=np.uint64)]).astype(np.uint32)
    assert np.array_equal(out, exp)


def _ka_model(recs: np.ndarray, n: int):
    """CPU model of K-a from its definition: per tile counts of byte 0, exclusive offsets, hist16."""
    r = recs.reshape(n, 100)
    T = -(-n // TILE)
    cnt = np.zeros((256, T), dtype=np.uint32)
    for t in range(T):
        b0 = r[t * TILE:(t + 1) * TILE, 0]
        cnt[:, t] = np.bincount(b0, minlength=256)
    lo = np.zeros((T, 256), dtype=np.uint32)
    lo[:, 1:] = np.cumsum(cnt.T, axis=1)[:, :-1]
    p16 = (r[:, 0].astype(np.uint32) << 8) | r[:, 1]
    hist16 = np.bincount(p16, minlength=65536).astype(np.uint32)
    return cnt, lo, hist16


@pytest.mark.parametrize("form", [1, 2, 0])
@pytest.mark.parametrize("n,dist", [(1, "uniform"), (3, "skewed"), (4095, "uniform"), (4097, "skewed"),
                                    (4098, "uniform"), (70_001, "uniform"), (300_007, "skewed"),
                                    (200_000, "all_equal")])
def test_ka_tile_sort_matches_model(form, n, dist):
    recs = gen.records(n, seed=n + form, dist=dist)
    T = -(-n // TILE)
    x = torch.from_numpy(recs).cuda()
    k1 = torch.empty(n, dtype=torch.int64, device="cuda")
    w = torch.empty(n, dtype=torch.int32, device="cuda")
    cnt = torch.empty(256 * T, dtype=torch.int32, device="cuda")
    lo = torch.empty(T * 256, dtype=torch.int32, device="cuda")
    h16 = torch.empty(65536, dtype=torch.int32, device="cuda")
    ley.ley_test_tile_sort(x, n, k1, w, cnt, lo, h16, stream_form=form)
    ecnt, elo, eh16 = _ka_model(recs, n)
    assert np.array_equal(cnt.cpu().numpy().view(np.uint32).reshape(256, T), ecnt)
    assert np.array_equal(lo.cpu().numpy().view(np.uint32).reshape(T, 256), elo)
    assert np.array_equal(h16.cpu().numpy().view(np.uint32), eh16)
    # pairs: each tile's byte-0 runs hold exactly that tile's (key bytes 1..9, local index) of that byte
    K1 = k1.cpu().numpy().view(np.uint64)
    W = w.cpu().numpy().view(np.uint32)
    r = recs.reshape(n, 100)
    for t in sorted({0, T // 2, T - 1}):
        base = t * TILE
        m = min(TILE, n - base)
        for b in np.nonzero(ecnt[:, t])[0][:40]:
            s0, c = elo[t, b], ecnt[b, t]
            got = sorted(zip(K1[base + s0: base + s0 + c].tolist(), W[base + s0: base + s0 + c].tolist()))
            loc = np.nonzero(r[base:base + m, 0] == b)[0]
            exp = []
            for i in loc:
                key = r[base + i, :10]
                k = int.from_bytes(bytes(key[1:9]), "big")
                exp.append((k, (int(key[9]) << 24) | int(i)))
            assert got == sorted(exp), (t, b)
