"""XCHECK — TEST INFRASTRUCTURE ONLY. ctypes glue for oracle/libxcheck.so, the
independent CSR graph-pattern counters of oracle/xcheck.cpp (triangles,
oriented 4-cliques, walk counts) that cross-check the Free Join oracle."""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libxcheck.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2301_10841_b200/build.py")
        L = C.CDLL(LIB_PATH)
        P, U64 = C.c_void_p, C.c_uint64
        L.xc_clique4.restype = C.c_int
        L.xc_clique4.argtypes = [P, P, U64, C.c_int, C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)]
        L.xc_triangles.restype = C.c_int
        L.xc_triangles.argtypes = [P, P, U64, C.c_int, C.c_uint32, C.c_uint32, C.POINTER(U64), C.POINTER(U64),
                                   C.POINTER(U64)]
        L.xc_walks.restype = C.c_int
        L.xc_walks.argtypes = [P, P, U64, C.c_int, P, C.c_int, C.c_int, P]
        _lib = L
    return _lib


def _threads(n):
    return n or os.cpu_count() or 1


def _count(fn, src, dst, nthreads, *extra):
    s = np.ascontiguousarray(src, dtype=np.int32)
    d = np.ascontiguousarray(dst, dtype=np.int32)
    lo, hi, ck = C.c_uint64(), C.c_uint64(), C.c_uint64()
    fn(s.ctypes.data, d.ctypes.data, len(s), _threads(nthreads), *extra, C.byref(lo), C.byref(hi), C.byref(ck))
    return {"count": (hi.value << 64) | lo.value, "checksum": ck.value}


def triangles(src, dst, nthreads=0, nparts=1, part=0):
    """Q(a,b,c) :- E(a,b),E(b,c),E(a,c): count and checksum (head order a,b,c);
    with nparts > 1 only the outputs whose a is in first-variable partition `part`."""
    return _count(lib().xc_triangles, src, dst, nthreads, nparts, part)


def clique4(src, dst, nthreads=0):
    """Oriented 4-cliques a->b,a->c,b->c,a->d,b->d,c->d: count and checksum (a,b,c,d)."""
    return _count(lib().xc_clique4, src, dst, nthreads)


def walks(src, dst, length, mods=(), nthreads=0):
    """Number of `length`-edge walks: [mod 2^64] + [mod p for p in mods]."""
    s = np.ascontiguousarray(src, dtype=np.int32)
    d = np.ascontiguousarray(dst, dtype=np.int32)
    m = np.asarray(mods, dtype=np.uint64)
    out = np.zeros(1 + len(mods), dtype=np.uint64)
    lib().xc_walks(s.ctypes.data, d.ctypes.data, len(s), length, m.ctypes.data if len(m) else None, len(m),
                   _threads(nthreads), out.ctypes.data)
    return [int(x) for x in out]
