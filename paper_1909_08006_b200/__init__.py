"""paper_1909_08006_b200 — B200-native (sm_100a) stable MSB radix sort of 100-byte records.

The hot path of Leyenda (arXiv 1909.08006, §3.1-§3.2) as hand-written CUDA behind a C ABI
(``include/leyenda.h``, ``libleyenda.so``). This module is the thin Python binding: the same names as the
C entry points, argument marshalling only. Every step of the sort runs in the library's kernels; there is
no CPU fallback — importing fails loudly if the native library is missing.

Pointer arguments accept a ``torch.Tensor`` (its ``data_ptr()``), a numpy array (its buffer address) or a
plain integer address. ``stream`` accepts a ``torch.cuda.Stream``, a raw ``cudaStream_t`` integer or
``None`` (legacy default stream).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LEY_LIBRARY_OVERRIDE: load a variant build of the same library (tools/build_variant.sh, A/B timing only)
_LIB_PATH = os.environ.get("LEY_LIBRARY_OVERRIDE") or os.path.join(_HERE, "libleyenda.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no fallback implementation)")

_lib = ctypes.CDLL(_LIB_PATH)

LEY_OK = 0
LEY_ERR_INVALID_ARGUMENT = 1
LEY_ERR_UNSUPPORTED = 2
LEY_ERR_BUDGET = 3
LEY_ERR_TOO_LARGE = 4
LEY_ERR_CAPACITY = 5
LEY_ERR_CUDA = 6
LEY_ERR_NCCL = 7
STATUS_NAMES = {0: "LEY_OK", 1: "LEY_ERR_INVALID_ARGUMENT", 2: "LEY_ERR_UNSUPPORTED", 3: "LEY_ERR_BUDGET",
                4: "LEY_ERR_TOO_LARGE", 5: "LEY_ERR_CAPACITY", 6: "LEY_ERR_CUDA", 7: "LEY_ERR_NCCL"}
RECORD_BYTES = 100
KEY_BYTES = 10
MAX_RECORDS = 0xFFFFFFFE

EXPORTED_SYMBOLS = ("ley_sort", "ley_sort_perm", "ley_last_error", "ley_comm_get_unique_id", "ley_comm_init",
                    "ley_sort_dist", "ley_comm_destroy", "ley_plan_query", "ley_set_option", "ley_get_option",
                    "ley_stage_times", "ley_release_cache", "ley_version", "ley_sort_dist_loopback",
                    "ley_dist_plan_splitters", "ley_dist_bin_dest_counts", "ley_dist_plan_exchange",
                    "ley_dist_dest_offsets", "ley_test_shared_scratch", "ley_test_shared_scratch_close",
                    "ley_sort_submit", "ley_sort_drain", "ley_test_scan_excl", "ley_test_tile_sort", "ley_device_bytes")


class ley_plan_info(ctypes.Structure):
    _fields_ = [("n_records", ctypes.c_uint64), ("tile_records", ctypes.c_uint64), ("tiles", ctypes.c_uint64),
                ("chunk_records", ctypes.c_uint64), ("internal_scratch", ctypes.c_uint64),
                ("staged_bytes", ctypes.c_uint64), ("host_path", ctypes.c_int32), ("run_records", ctypes.c_uint64),
                ("runs", ctypes.c_uint64), ("resident_bytes", ctypes.c_uint64)]


_u64, _u32, _i32, _i64, _vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
_lib.ley_sort.argtypes = [_vp, _vp, _u64, _u32, _u32, _u64, _vp]
_lib.ley_sort.restype = _i32
_lib.ley_sort_perm.argtypes = [_vp, _vp, _vp, _u64, _u32, _u32, _u64, _vp]
_lib.ley_sort_perm.restype = _i32
_lib.ley_sort_submit.argtypes = [_vp, _vp, _u64, _u32, _u32, _u64, _vp]
_lib.ley_sort_submit.restype = _i32
_lib.ley_sort_drain.argtypes = []
_lib.ley_sort_drain.restype = _i32
_lib.ley_test_scan_excl.argtypes = [_vp, _vp, _u64, _vp]
_lib.ley_test_scan_excl.restype = _i32
_lib.ley_test_tile_sort.argtypes = [_vp, _u64, _vp, _vp, _vp, _vp, _vp, _i32, _vp]
_lib.ley_test_tile_sort.restype = _i32
_lib.ley_device_bytes.argtypes = [ctypes.POINTER(_u64), ctypes.POINTER(_u64), _i32]
_lib.ley_device_bytes.restype = _i32
_lib.ley_last_error.argtypes = []
_lib.ley_last_error.restype = ctypes.c_char_p
_lib.ley_comm_get_unique_id.argtypes = [_vp]
_lib.ley_comm_get_unique_id.restype = _i32
_lib.ley_comm_init.argtypes = [ctypes.POINTER(_vp), _i32, _i32, _vp, _i32]
_lib.ley_comm_init.restype = _i32
_lib.ley_sort_dist.argtypes = [_vp, _vp, _u64, _vp, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64), _u32, _u32,
                               _u64, _vp]
_lib.ley_sort_dist.restype = _i32
_lib.ley_comm_destroy.argtypes = [_vp]
_lib.ley_comm_destroy.restype = _i32
_lib.ley_plan_query.argtypes = [_u64, _u64, ctypes.POINTER(ley_plan_info)]
_lib.ley_plan_query.restype = _i32
_lib.ley_set_option.argtypes = [ctypes.c_char_p, _i64]
_lib.ley_set_option.restype = _i32
_lib.ley_get_option.argtypes = [ctypes.c_char_p, ctypes.POINTER(_i64)]
_lib.ley_get_option.restype = _i32
_lib.ley_stage_times.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float), _i32,
                                 ctypes.POINTER(_i32)]
_lib.ley_stage_times.restype = _i32
_lib.ley_release_cache.argtypes = [_i32]
_lib.ley_release_cache.restype = _i32
_lib.ley_version.argtypes = []
_lib.ley_version.restype = _u32
_pu64 = ctypes.POINTER(_u64)
_lib.ley_sort_dist_loopback.argtypes = [_i32, ctypes.POINTER(_vp), _pu64, ctypes.POINTER(_vp), _pu64, _pu64, _pu64,
                                        _u32, _u32, _u64, _vp]
_lib.ley_sort_dist_loopback.restype = _i32
_lib.ley_dist_plan_splitters.argtypes = [_pu64, _u64, _i32, ctypes.POINTER(_u32), _pu64, _pu64]
_lib.ley_dist_plan_splitters.restype = _i32
_lib.ley_dist_bin_dest_counts.argtypes = [_pu64, ctypes.POINTER(_u32), _i32, _pu64]
_lib.ley_dist_bin_dest_counts.restype = None
_lib.ley_dist_plan_exchange.argtypes = [_pu64, _i32, _i32, _pu64, _pu64, _pu64, _pu64, _pu64]
_lib.ley_dist_plan_exchange.restype = None
_lib.ley_dist_dest_offsets.argtypes = [_pu64, _i32, _i32, _pu64]
_lib.ley_dist_dest_offsets.restype = None
_lib.ley_test_shared_scratch.argtypes = [ctypes.c_char_p, _u64, _i32, ctypes.POINTER(_vp)]
_lib.ley_test_shared_scratch.restype = _i32
_lib.ley_test_shared_scratch_close.argtypes = [_vp, _u64, ctypes.c_char_p]
_lib.ley_test_shared_scratch_close.restype = None


class LeyendaError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.ley_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")


def _addr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)!r}")


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    if hasattr(s, "cuda_stream"):
        return s.cuda_stream
    raise TypeError(f"not a stream: {type(s)!r}")


def _check(st: int, where: str, raise_on_error: bool):
    if st != LEY_OK and raise_on_error:
        raise LeyendaError(st, where)
    return st


def ley_sort(in_, out, n_records: int, record_bytes: int = RECORD_BYTES, key_bytes: int = KEY_BYTES,
             device_budget_bytes: int = 0, stream=None, raise_on_error: bool = True) -> int:
    """C: ley_sort(in, out, n_records, record_bytes, key_bytes, device_budget_bytes, stream)."""
    st = _lib.ley_sort(_addr(in_), _addr(out), n_records, record_bytes, key_bytes, device_budget_bytes, _stream(stream))
    return _check(st, "ley_sort", raise_on_error)


def ley_sort_submit(in_, out, n_records: int, record_bytes: int = RECORD_BYTES, key_bytes: int = KEY_BYTES,
                    device_budget_bytes: int = 0, stream=None, raise_on_error: bool = True) -> int:
    """C: ley_sort_submit(in, out, n_records, ...): pipelined sort of pinned host records (see leyenda.h)."""
    st = _lib.ley_sort_submit(_addr(in_), _addr(out), n_records, record_bytes, key_bytes, device_budget_bytes,
                              _stream(stream))
    return _check(st, "ley_sort_submit", raise_on_error)


def ley_sort_drain(raise_on_error: bool = True) -> int:
    """C: ley_sort_drain(): wait for every submitted sort on the current device."""
    return _check(_lib.ley_sort_drain(), "ley_sort_drain", raise_on_error)


def ley_sort_perm(in_, out, perm, n_records: int, record_bytes: int = RECORD_BYTES, key_bytes: int = KEY_BYTES,
                  device_budget_bytes: int = 0, stream=None, raise_on_error: bool = True) -> int:
    """C: ley_sort_perm(in, out, perm, n_records, ...); perm: u32[n_records]."""
    st = _lib.ley_sort_perm(_addr(in_), _addr(out), _addr(perm), n_records, record_bytes, key_bytes,
                            device_budget_bytes, _stream(stream))
    return _check(st, "ley_sort_perm", raise_on_error)


def ley_last_error() -> str:
    return _lib.ley_last_error().decode(errors="replace")


def ley_plan_query(n_records: int, device_budget_bytes: int = 0) -> dict:
    info = ley_plan_info()
    st = _lib.ley_plan_query(n_records, device_budget_bytes, ctypes.byref(info))
    _check(st, "ley_plan_query", True)
    return {name: getattr(info, name) for name, _ in ley_plan_info._fields_}


def ley_set_option(name: str, value: int) -> None:
    _check(_lib.ley_set_option(name.encode(), int(value)), "ley_set_option", True)


def ley_get_option(name: str) -> int:
    v = ctypes.c_int64()
    _check(_lib.ley_get_option(name.encode(), ctypes.byref(v)), "ley_get_option", True)
    return v.value


def ley_stage_times(max_stages: int = 64):
    """[(stage name, ms)] of the last call on this thread (with option "profile" = 1), and its launch count."""
    names = (ctypes.c_char_p * max_stages)()
    ms = (ctypes.c_float * max_stages)()
    launches = ctypes.c_int()
    k = _lib.ley_stage_times(names, ms, max_stages, ctypes.byref(launches))
    return [(names[i].decode(), ms[i]) for i in range(k)], launches.value


def ley_release_cache(device: int = -1) -> None:
    _lib.ley_release_cache(device)


def ley_version() -> tuple[int, int]:
    v = _lib.ley_version()
    return v >> 16, v & 0xFFFF


# ---------------------------------------------------------------- multi-GPU
def ley_comm_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.ley_comm_get_unique_id(buf), "ley_comm_get_unique_id", True)
    return bytes(buf)


def ley_comm_init(nranks: int, rank: int, unique_id: bytes, device: int) -> int:
    comm = ctypes.c_void_p()
    idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
    _check(_lib.ley_comm_init(ctypes.byref(comm), nranks, rank, idbuf, device), "ley_comm_init", True)
    return comm.value


def ley_sort_dist(comm: int, in_local, n_local: int, out_local, out_capacity_records: int,
                  record_bytes: int = RECORD_BYTES, key_bytes: int = KEY_BYTES, device_budget_bytes: int = 0,
                  stream=None):
    """Returns (n_out_local, out_global_offset)."""
    n_out = ctypes.c_uint64()
    off = ctypes.c_uint64()
    st = _lib.ley_sort_dist(comm, _addr(in_local), n_local, _addr(out_local), out_capacity_records,
                            ctypes.byref(n_out), ctypes.byref(off), record_bytes, key_bytes, device_budget_bytes,
                            _stream(stream))
    _check(st, "ley_sort_dist", True)
    return n_out.value, off.value


def ley_comm_destroy(comm: int) -> None:
    _check(_lib.ley_comm_destroy(comm), "ley_comm_destroy", True)


def ley_sort_dist_loopback(ins, n_locals, outs, caps, record_bytes: int = RECORD_BYTES, key_bytes: int = KEY_BYTES,
                           device_budget_bytes: int = 0, stream=None):
    """G logical ranks on the current device (test hook). Returns [(n_out, out_global_offset)] per rank."""
    G = len(ins)
    a_in = (_vp * G)(*[_addr(x) for x in ins])
    a_out = (_vp * G)(*[_addr(x) for x in outs])
    a_n = (_u64 * G)(*n_locals)
    a_cap = (_u64 * G)(*caps)
    n_out = (_u64 * G)()
    off = (_u64 * G)()
    st = _lib.ley_sort_dist_loopback(G, a_in, a_n, a_out, a_cap, n_out, off, record_bytes, key_bytes,
                                     device_budget_bytes, _stream(stream))
    _check(st, "ley_sort_dist_loopback", True)
    return [(n_out[i], off[i]) for i in range(G)]


def ley_dist_plan_splitters(global_hist16, n_total: int, nranks: int):
    """-> (bins, rank_in_bin, bin_first), each a list of nranks-1 ints."""
    h = (_u64 * 65536)(*[int(x) for x in global_hist16])
    k = max(nranks - 1, 1)
    bins, rho, first = (_u32 * k)(), (_u64 * k)(), (_u64 * k)()
    rc = _lib.ley_dist_plan_splitters(h, n_total, nranks, bins, rho, first)
    if rc:
        raise ValueError(f"ley_dist_plan_splitters failed ({rc})")
    return list(bins)[: nranks - 1], list(rho)[: nranks - 1], list(first)[: nranks - 1]


def ley_dist_bin_dest_counts(local_hist16, bins, nranks: int):
    h = (_u64 * 65536)(*[int(x) for x in local_hist16])
    b = (_u32 * max(len(bins), 1))(*bins)
    c = (_u64 * nranks)()
    _lib.ley_dist_bin_dest_counts(h, b, nranks, c)
    return list(c)


def ley_dist_plan_exchange(send_counts, nranks: int, rank: int):
    """send_counts: nranks x nranks [src][dst] -> dict(recv_counts, recv_offsets, send_offsets, n_out, out_offset)."""
    flat = [int(x) for row in send_counts for x in row]
    m = (_u64 * (nranks * nranks))(*flat)
    rc, ro, so = (_u64 * nranks)(), (_u64 * nranks)(), (_u64 * nranks)()
    n_out, off = _u64(), _u64()
    _lib.ley_dist_plan_exchange(m, nranks, rank, rc, ro, so, ctypes.byref(n_out), ctypes.byref(off))
    return dict(recv_counts=list(rc), recv_offsets=list(ro), send_offsets=list(so), n_out=n_out.value,
                out_offset=off.value)


def ley_dist_dest_offsets(send_counts, nranks: int, rank: int):
    """send_counts: nranks x nranks [src][dst] -> where this rank's run starts in each destination's buffer."""
    flat = [int(x) for row in send_counts for x in row]
    m = (_u64 * (nranks * nranks))(*flat)
    d = (_u64 * nranks)()
    _lib.ley_dist_dest_offsets(m, nranks, rank, d)
    return list(d)


def ley_test_shared_scratch(name: str, nbytes: int, create: bool) -> int:
    """Create/open + map the shared run scratch segment (host logic only); returns its address."""
    p = _vp()
    _check(_lib.ley_test_shared_scratch(name.encode(), nbytes, int(create), ctypes.byref(p)), "ley_test_shared_scratch",
           True)
    return p.value


def ley_test_shared_scratch_close(addr: int, nbytes: int, unlink_name: str | None = None) -> None:
    _lib.ley_test_shared_scratch_close(addr, nbytes, unlink_name.encode() if unlink_name else None)


def library_path() -> str:
    return _LIB_PATH


def ley_test_scan_excl(in_, out, m: int, stream=None) -> int:
    """C: ley_test_scan_excl(in, out, m, stream) — K-b alone (verification hook)."""
    return _check(_lib.ley_test_scan_excl(_addr(in_), _addr(out), m, _stream(stream)), "ley_test_scan_excl", True)


def ley_test_tile_sort(in_, n: int, k1, w, cnt, lo, hist16, stream_form: int = 1, stream=None) -> int:
    """C: ley_test_tile_sort(in, n, k1, w, cnt, lo, hist16, stream_form, stream) — K-a alone (verification hook)."""
    st = _lib.ley_test_tile_sort(_addr(in_), n, _addr(k1), _addr(w), _addr(cnt), _addr(lo), _addr(hist16),
                                 stream_form, _stream(stream))
    return _check(st, "ley_test_tile_sort", True)


def ley_device_bytes(reset_peak: bool = False) -> tuple[int, int]:
    """C: ley_device_bytes(&current, &peak, reset_peak) -> (current, peak) bytes held by the library."""
    cur, peak = _u64(), _u64()
    _check(_lib.ley_device_bytes(ctypes.byref(cur), ctypes.byref(peak), int(reset_peak)), "ley_device_bytes", True)
    return cur.value, peak.value
