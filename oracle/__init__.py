"""CPU oracle for the Leyenda record sort — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package. The product (``paper_1909_08006_b200``) never imports it and shares no code
with it. See ``oracle/oracle.cpp`` for the definition it implements and the passages it cites
(§3.1-§3.2, lines 50-106; BASELINE.json north_star).

Every function here is a thin ctypes wrapper over ``oracle/liboracle.so`` (built from ``oracle.cpp`` by
``build_native.build_oracle``) working on numpy uint8 arrays of shape (n*100,) or (n, 100).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

RECORD_BYTES = 100
KEY_BYTES = 10


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "oracle.cpp")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            import sys

            sys.path.insert(0, os.path.dirname(_HERE))
            from build_native import build_oracle

            build_oracle()
        lib = ctypes.CDLL(path)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        lib.oracle_sort.argtypes = [vp, vp, vp, u64, i32]
        lib.oracle_sort.restype = i32
        lib.oracle_sort_timed.argtypes = [vp, vp, u64, i32, ctypes.POINTER(ctypes.c_double)]
        lib.oracle_sort_timed.restype = i32
        lib.oracle_multiset_hash.argtypes = [vp, u64, ctypes.POINTER(u64), i32]
        lib.oracle_multiset_hash.restype = None
        lib.oracle_sequence_digest.argtypes = [vp, u64, u64, ctypes.POINTER(u64), i32]
        lib.oracle_sequence_digest.restype = None
        lib.oracle_sorted_digest.argtypes = [vp, u64, ctypes.POINTER(u64), i32]
        lib.oracle_sorted_digest.restype = i32
        lib.oracle_is_sorted.argtypes = [vp, u64]
        lib.oracle_is_sorted.restype = i32
        lib.oracle_certify.argtypes = [vp, vp, vp, u64]
        lib.oracle_certify.restype = u64
        lib.oracle_sort_kb.argtypes = [vp, vp, vp, u64, i32, i32]
        lib.oracle_sort_kb.restype = i32
        lib.oracle_certify_kb.argtypes = [vp, vp, vp, u64, i32]
        lib.oracle_certify_kb.restype = u64
        _LIB = lib
    return _LIB


def _flat(recs) -> np.ndarray:
    a = np.ascontiguousarray(recs, dtype=np.uint8).reshape(-1)
    if a.size % RECORD_BYTES:
        raise ValueError("record buffer size is not a multiple of 100 bytes")
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def sort(recs, threads: int = 0, want_perm: bool = True, key_bytes: int = 10):
    """Stable ascending sort of 100-byte records by the unsigned key = bytes [0, key_bytes) (ties by index).

    Returns (out, perm): out is a (n*100,) uint8 array, perm[j] the input index of output record j.
    key_bytes = 10 (the paper's records) uses the (key, pointer) tuple sort; other sizes (P:164
    flexible key sizes, 1..100) compare the records themselves.
    """
    a = _flat(recs)
    n = a.size // RECORD_BYTES
    out = np.empty_like(a)
    perm = np.empty(n, dtype=np.uint32) if want_perm else None
    pp = _ptr(perm) if perm is not None else None
    if key_bytes == 10:
        rc = _lib().oracle_sort(_ptr(a), _ptr(out), pp, n, threads)
    else:
        rc = _lib().oracle_sort_kb(_ptr(a), _ptr(out), pp, n, key_bytes, threads)
    if rc:
        raise ValueError(f"oracle_sort: n or key_bytes out of range (rc {rc})")
    return out, perm


def sort_timed(recs, threads: int = 0):
    """Sort and return (out, (extract_s, sort_s, gather_s)) — the CPU baseline's stage breakdown."""
    a = _flat(recs)
    n = a.size // RECORD_BYTES
    out = np.empty_like(a)
    secs = (ctypes.c_double * 3)()
    rc = _lib().oracle_sort_timed(_ptr(a), _ptr(out), n, threads, secs)
    if rc:
        raise ValueError("oracle_sort_timed: n out of range")
    return out, (secs[0], secs[1], secs[2])


def multiset_hash(recs, threads: int = 0) -> int:
    """Permutation-invariant 128-bit digest (sum of per-record hashes mod 2^128)."""
    a = _flat(recs)
    out = (ctypes.c_uint64 * 2)()
    _lib().oracle_multiset_hash(_ptr(a), a.size // RECORD_BYTES, out, threads)
    return out[0] | (out[1] << 64)


def sequence_digest(recs, j0: int = 0, threads: int = 0) -> int:
    """Order-dependent 128-bit digest of a record sequence starting at global position j0.

    Digests of consecutive slices add (mod 2^128) to the digest of their concatenation."""
    a = _flat(recs)
    out = (ctypes.c_uint64 * 2)()
    _lib().oracle_sequence_digest(_ptr(a), a.size // RECORD_BYTES, j0, out, threads)
    return out[0] | (out[1] << 64)


def sorted_digest(recs, threads: int = 0) -> int:
    """sequence_digest of the oracle's sorted output, without materialising that output."""
    a = _flat(recs)
    out = (ctypes.c_uint64 * 2)()
    rc = _lib().oracle_sorted_digest(_ptr(a), a.size // RECORD_BYTES, out, threads)
    if rc:
        raise ValueError("oracle_sorted_digest: n out of range")
    return out[0] | (out[1] << 64)


def is_sorted(recs) -> bool:
    a = _flat(recs)
    return bool(_lib().oracle_is_sorted(_ptr(a), a.size // RECORD_BYTES))


def certify(inp, out, perm, key_bytes: int = 10) -> int:
    """0 if (perm is a permutation, out[j] == in[perm[j]], (key, perm) strictly increasing); else
    1 + first failing position (n + 1 for a non-permutation)."""
    a, b = _flat(inp), _flat(out)
    p = np.ascontiguousarray(perm, dtype=np.uint32)
    n = a.size // RECORD_BYTES
    if b.size != a.size or p.size != n:
        raise ValueError("certify: size mismatch")
    if key_bytes == 10:
        return int(_lib().oracle_certify(_ptr(a), _ptr(b), _ptr(p), n))
    return int(_lib().oracle_certify_kb(_ptr(a), _ptr(b), _ptr(p), n, key_bytes))


def mod128(x: int) -> int:
    return x & ((1 << 128) - 1)
