"""ORACLE GENERATORS — TEST / BASELINE INFRASTRUCTURE ONLY. ctypes glue for
oracle/libogen.so (oracle/gen.cpp): an independent implementation of the
seeded config inputs, so the reference arm never loads a product library."""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libogen.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2301_10841_b200/build.py")
        L = C.CDLL(LIB_PATH)
        P, U64 = C.c_void_p, C.c_uint64
        L.og_uniform.argtypes = [U64, C.c_uint32, U64, U64, P]
        L.og_zipf.argtypes = [U64, C.c_uint32, U64, U64, C.c_double, P]
        L.og_zipf.restype = C.c_int
        L.og_rmat.argtypes = [U64, C.c_int, U64, C.c_double, C.c_double, C.c_double, P, P]
        L.og_rmat.restype = C.c_int
        L.og_orient.argtypes = [U64, P, P, U64, P, P]
        L.og_orient.restype = C.c_int64
        _lib = L
    return _lib


def uniform(seed, col, n, domain):
    out = np.empty(max(n, 1), dtype=np.int32)
    lib().og_uniform(seed, col, n, domain, out.ctypes.data)
    return out[:n]


def zipf(seed, stream, n, k, s):
    out = np.empty(max(n, 1), dtype=np.int32)
    if lib().og_zipf(seed, stream, n, k, s, out.ctypes.data) != 0:
        raise ValueError("zipf: empty domain")
    return out[:n]


def rmat(seed, scale, m, a=0.57, b=0.19, c=0.19):
    s = np.empty(max(m, 1), dtype=np.int32)
    d = np.empty(max(m, 1), dtype=np.int32)
    if lib().og_rmat(seed, scale, m, a, b, c, s.ctypes.data, d.ctypes.data) != 0:
        raise ValueError("rmat: scale must be 1..31")
    return [s[:m], d[:m]]


def orient(seed, src, dst):
    n = len(src)
    os_ = np.empty(max(n, 1), dtype=np.int32)
    od = np.empty(max(n, 1), dtype=np.int32)
    s = np.ascontiguousarray(src, dtype=np.int32)
    d = np.ascontiguousarray(dst, dtype=np.int32)
    k = lib().og_orient(seed, s.ctypes.data, d.ctypes.data, n, os_.ctypes.data, od.ctypes.data)
    return [os_[:k].copy(), od[:k].copy()]
