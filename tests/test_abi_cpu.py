"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports every symbol that
include/leyenda.h declares, validates arguments before touching CUDA, and plans (host-only)."""
import os
import re

import pytest

import build_native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ley():
    build_native.build_leyenda()
    import paper_1909_08006_b200 as ley

    return ley


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "leyenda.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ley_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(ley):
    import ctypes

    declared = _declared_symbols()
    assert len(declared) >= 13
    lib = ctypes.CDLL(ley.library_path())
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(ley.EXPORTED_SYMBOLS)


def test_version(ley):
    assert ley.ley_version() == (1, 1)


def test_validation_before_cuda(ley):
    # records other than 100 bytes or keys outside 1..100 bytes -> UNSUPPORTED, even
    # with n = 0
    assert ley.ley_sort(0, 0, 0, 99, 10, raise_on_error=False) == ley.LEY_ERR_UNSUPPORTED
    assert "record_bytes must be 100" in ley.ley_last_error()
    for kb in (0, 101):
        assert ley.ley_sort(0, 0, 0, 100, kb, raise_on_error=False) == ley.LEY_ERR_UNSUPPORTED
    # a shorter key is valid: the NULL pointers are what is wrong
    assert ley.ley_sort(0, 0, 10, 100, 8, raise_on_error=False) == ley.LEY_ERR_INVALID_ARGUMENT
    # n = 0 is OK and touches nothing
    assert ley.ley_sort(0, 0, 0, raise_on_error=False) == ley.LEY_OK
    assert ley.ley_last_error() == ""
    # n > 2^32 - 2 -> TOO_LARGE
    assert ley.ley_sort(16, 4096, 2**32 - 1, raise_on_error=False) == ley.LEY_ERR_TOO_LARGE
    # NULL with n > 0, misalignment, overlap -> INVALID_ARGUMENT
    assert ley.ley_sort(0, 4096, 5, raise_on_error=False) == ley.LEY_ERR_INVALID_ARGUMENT
    assert ley.ley_sort(4100, 1 << 20, 5, raise_on_error=False) == ley.LEY_ERR_INVALID_ARGUMENT
    assert ley.ley_sort(1 << 20, (1 << 20) + 256, 5, raise_on_error=False) == ley.LEY_ERR_INVALID_ARGUMENT
    assert "overlap" in ley.ley_last_error()


def test_plan_query(ley):
    p = ley.ley_plan_query(100_000_000)
    assert p["tiles"] == (100_000_000 + 4095) // 4096
    assert p["host_path"] == 0 and p["runs"] == 1
    # internal scratch ~ 12 + 12 + 4 bytes/record plus per-tile tables (SURVEY Appendix B layout)
    assert 28e8 < p["internal_scratch"] < 32e8
    assert p["staged_bytes"] >= p["internal_scratch"] + 2 * 100 * 100_000_000
    # 60 GB under a 4 GB budget -> external, runs of bounded size (BASELINE.json configs[4])
    e = ley.ley_plan_query(600_000_000, 4 << 30)
    assert e["host_path"] == 1
    assert 1 <= e["run_records"] < 600_000_000
    assert e["runs"] == -(-600_000_000 // e["run_records"])
    assert 200 * e["run_records"] + ley.ley_plan_query(e["run_records"])["internal_scratch"] <= 4 << 30
    # between the two: the input fits but input + output do not -> path 2 (resident input, streamed
    # output); its device bytes = scratch + 100 n (input) + 4 n (perm) + two output windows
    r = ley.ley_plan_query(200_000_000, 30_000_000_000)
    assert r["host_path"] == 2 and r["resident_bytes"] <= 30_000_000_000 < r["staged_bytes"]
    assert r["resident_bytes"] == (r["internal_scratch"] + 100 * 200_000_000 + 4 * 200_000_000 +
                                   2 * 100 * (1 << 21))
    assert ley.ley_plan_query(200_000_000, r["resident_bytes"] - 1)["host_path"] == 1
    ley.ley_set_option("resident_path", 0)
    try:
        assert ley.ley_plan_query(200_000_000, 30_000_000_000)["host_path"] == 1
    finally:
        ley.ley_set_option("resident_path", 1)
    with pytest.raises(ley.LeyendaError):
        ley.ley_plan_query(2**32)


def test_options(ley):
    assert ley.ley_get_option("smem_tier_max") == 16384
    ley.ley_set_option("kd_insert_max", 8)
    assert ley.ley_get_option("kd_insert_max") == 8
    ley.ley_set_option("kd_insert_max", 16)
    with pytest.raises(ley.LeyendaError):
        ley.ley_set_option("warp_tier_max", 33)
    with pytest.raises(ley.LeyendaError):
        ley.ley_set_option("no_such_option", 1)


def test_documented_options_exist(ley):
    """Every option the header documents can be read (and only real names can): the header's option list
    and the library's registry agree."""
    import re

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "leyenda.h")).read()
    block = hdr[hdr.index("Integer options"):hdr.index("ley_status ley_set_option")]
    names = re.findall(r'^ \*   "([a-z_0-9]+)"', block, flags=re.M)
    assert len(names) >= 15
    for nm in names:
        ley.ley_get_option(nm)  # raises on an unknown name
    with pytest.raises(ley.LeyendaError):
        ley.ley_get_option("no_such_option")
