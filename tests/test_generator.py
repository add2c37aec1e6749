"""Generator tests (-m "not gpu"): determinism, slicing and the BASELINE.json configs[2] statistics.

The generator is input generation only (gen/gen_core.h); these tests pin that the
synthetic inputs have the shapes and distributions the configs name."""
import math

import numpy as np

import gen


def test_deterministic_and_sliceable():
    a = gen.records(5000, seed=4)
    b = gen.records(5000, seed=4)
    assert np.array_equal(a, b)
    c = gen.records(1000, seed=4, i0=2500)
    assert np.array_equal(a[2500 * 100: 3500 * 100], c)
    assert not np.array_equal(gen.records(10, seed=5), a[:1000])


def test_uniform_first_byte_chi2():
    k = gen.keys(256 * 400, seed=1)
    for byte in (0, 1, 9):
        counts = np.bincount(k[:, byte], minlength=256)
        exp = k.shape[0] / 256
        chi2 = float(((counts - exp) ** 2 / exp).sum())
        # 255 dof: mean 255, sd ~22.6; 6 sd bound
        assert chi2 < 255 + 6 * math.sqrt(2 * 255), (byte, chi2)


def test_skewed_zipf_and_byte1():
    n = 400000
    k = gen.keys(n, seed=2, dist="skewed")
    zt = gen.zipf_table()
    probs = [zt[0] / 2**64] + [(zt[v] - zt[v - 1]) / 2**64 for v in range(1, 256)]
    h = sum(r ** -1.2 for r in range(1, 257))
    for v in range(8):
        assert abs(probs[v] - (v + 1) ** -1.2 / h) < 1e-12
    assert abs(probs[0] - 0.2536) < 1e-3 and abs(sum(probs[:8]) - 0.5917) < 1e-3
    counts = np.bincount(k[:, 0], minlength=256)
    for v in range(4):  # duplicates copy keys with the same distribution, so frequencies still hold
        p = probs[v]
        assert abs(counts[v] / n - p) < 6 * math.sqrt(p * (1 - p) / n), v
    assert k[:, 1].max() <= 7


def test_skewed_duplicates():
    seed, n = 2, 200000
    k = gen.keys(n, seed=seed, dist="skewed")
    srcs = [(i, gen.dup_source(seed, i)) for i in range(n)]
    dups = [(i, s) for i, s in srcs if s is not None]
    p = 0.02
    assert abs(len(dups) - p * n) < 5 * math.sqrt(n * p * (1 - p))
    assert gen.dup_source(seed, 0) is None
    for i, s in dups[:5000]:
        assert s < i
        assert bytes(k[i]) == bytes(k[s])


def test_edge_distributions():
    n = 2000
    assert len({bytes(x) for x in gen.keys(n, 1, "all_equal")}) == 1
    assert len({bytes(x) for x in gen.keys(n, 1, "three_keys")}) == 3
    s = [bytes(x) for x in gen.keys(n, 1, "sorted")]
    assert all(s[i] < s[i + 1] for i in range(n - 1))
    r = [bytes(x) for x in gen.keys(n, 1, "reverse")]
    assert all(r[i] > r[i + 1] for i in range(n - 1))
    p = gen.keys(n, 1, "prefix2")
    assert (p[:, 0] == 0xAB).all() and (p[:, 1] == 0xCD).all()
    b9 = gen.keys(n, 1, "byte9")
    assert (b9[:, :9] == b9[0, :9]).all() and len(set(b9[:, 9].tolist())) > 200
    a = gen.keys(n, 1, "ascii")
    assert a.min() >= 0x20 and a.max() <= 0x7E
    assert len(np.unique(a[:, 0])) == 95  # all 95 printable values occur as a first byte
    r = gen.records(n, 1, "ascii").reshape(n, 100)
    assert r[:, :98].min() >= 0x20 and r[:, :98].max() <= 0x7E
    assert (r[:, 98] == 13).all() and (r[:, 99] == 10).all()  # CR LF line ends (P:126 ASCII set)
    t = gen.keys(n, 1, "tiny_alphabet")
    assert set(np.unique(t).tolist()) <= {0, 1, 255}
