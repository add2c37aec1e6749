"""Seeded synthetic 100-byte record generator — input generation only.

Shared by the oracle tests and the GPU tests/bench; it holds none of the sort's arithmetic.
``records(...)`` runs on the host (OpenMP, ``gen/libleygen_host.so``); ``records_cuda(...)`` is the CUDA
twin (``gen/libleygen_cuda.so``) that writes straight into device memory. Both compile ``gen_core.h``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST = None
_CUDA = None

UNIFORM, SKEWED, ALL_EQUAL, THREE_KEYS, SORTED, REVERSE, PREFIX2, BYTE9, ASCII, TINY_ALPHABET = range(10)
DIST_NAMES = {
    "uniform": UNIFORM,
    "skewed": SKEWED,
    "all_equal": ALL_EQUAL,
    "three_keys": THREE_KEYS,
    "sorted": SORTED,
    "reverse": REVERSE,
    "prefix2": PREFIX2,
    "byte9": BYTE9,
    "ascii": ASCII,
    "tiny_alphabet": TINY_ALPHABET,
}


def _ensure_built(kind: str):
    import sys

    sys.path.insert(0, os.path.dirname(_HERE))
    import build_native

    if kind == "host":
        build_native.build_gen_host()
    else:
        build_native.build_gen_cuda()


def _host():
    global _HOST
    if _HOST is None:
        path = os.path.join(_HERE, "libleygen_host.so")
        srcs = [os.path.join(_HERE, f) for f in ("gen.cpp", "gen_core.h")]
        if not os.path.exists(path) or os.path.getmtime(path) < max(os.path.getmtime(s) for s in srcs):
            _ensure_built("host")
        lib = ctypes.CDLL(path)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        lib.gen_records.argtypes = [vp, u64, u64, u64, i32, i32]
        lib.gen_records.restype = None
        lib.gen_keys.argtypes = [vp, u64, u64, u64, i32, i32]
        lib.gen_keys.restype = None
        lib.gen_build_zipf.argtypes = [ctypes.POINTER(u64)]
        lib.gen_build_zipf.restype = None
        lib.gen_dup_source.argtypes = [u64, u64]
        lib.gen_dup_source.restype = u64
        _HOST = lib
    return _HOST


def _cuda():
    global _CUDA
    if _CUDA is None:
        path = os.path.join(_HERE, "libleygen_cuda.so")
        srcs = [os.path.join(_HERE, f) for f in ("gen_cuda.cu", "gen.cpp", "gen_core.h")]
        if not os.path.exists(path) or os.path.getmtime(path) < max(os.path.getmtime(s) for s in srcs):
            _ensure_built("cuda")
        lib = ctypes.CDLL(path)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        lib.gen_records_cuda.argtypes = [vp, u64, u64, u64, i32, vp]
        lib.gen_records_cuda.restype = i32
        _CUDA = lib
    return _CUDA


def _dist(d) -> int:
    return DIST_NAMES[d] if isinstance(d, str) else int(d)


def records(n: int, seed: int, dist="uniform", i0: int = 0, threads: int = 0) -> np.ndarray:
    """Records [i0, i0+n) as a flat (n*100,) uint8 array."""
    out = np.empty(n * 100, dtype=np.uint8)
    if n:
        _host().gen_records(out.ctypes.data_as(ctypes.c_void_p), i0, n, seed, _dist(dist), threads)
    return out


def keys(n: int, seed: int, dist="uniform", i0: int = 0, threads: int = 0) -> np.ndarray:
    """Only the keys of records [i0, i0+n), shape (n, 10)."""
    out = np.empty(n * 10, dtype=np.uint8)
    if n:
        _host().gen_keys(out.ctypes.data_as(ctypes.c_void_p), i0, n, seed, _dist(dist), threads)
    return out.reshape(n, 10)


def zipf_table() -> list[int]:
    zt = (ctypes.c_uint64 * 256)()
    _host().gen_build_zipf(zt)
    return list(zt)


def dup_source(seed: int, i: int):
    s = _host().gen_dup_source(seed, i)
    return None if s == (1 << 64) - 1 else s


def records_cuda(dev_ptr: int, n: int, seed: int, dist="uniform", i0: int = 0, stream: int = 0) -> None:
    """Write records [i0, i0+n) into device memory at dev_ptr (4-byte aligned). Synchronises `stream`."""
    rc = _cuda().gen_records_cuda(ctypes.c_void_p(dev_ptr), i0, n, seed, _dist(dist), ctypes.c_void_p(stream))
    if rc:
        raise RuntimeError(f"gen_records_cuda failed (rc={rc})")
