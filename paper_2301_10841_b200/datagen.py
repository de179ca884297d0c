"""Seeded synthetic inputs (ctypes over libfjgen.so, see csrc/datagen.cpp).

Generated arrays are cached as .npy files under $FJG_DATA_CACHE
(default /tmp/fjg_data) keyed by every generator parameter; a cache miss just
regenerates, so nothing depends on the cache surviving between GPU calls.
"""
import ctypes as C
import hashlib
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfjgen.so")
_lib = None

M = 1 << 20  # "M" of BASELINE.json configs (SURVEY.md §8 config shorthand)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2301_10841_b200/build.py")
        L = C.CDLL(LIB_PATH)
        P, U64 = C.c_void_p, C.c_uint64
        L.fjgen_uniform.argtypes = [U64, C.c_uint32, U64, U64, P]
        L.fjgen_zipf.argtypes = [U64, C.c_uint32, U64, U64, C.c_double, P]
        L.fjgen_zipf.restype = C.c_int
        L.fjgen_rmat.argtypes = [U64, C.c_int, U64, C.c_double, C.c_double, C.c_double, P, P]
        L.fjgen_rmat.restype = C.c_int
        L.fjgen_orient.argtypes = [U64, P, P, U64, P, P]
        L.fjgen_orient.restype = C.c_int64
        L.fjgen_last_error.restype = C.c_char_p
        L.fjgen_rmat_device.argtypes = [C.c_int, U64, C.c_int, U64, C.c_double, C.c_double, C.c_double, P, P]
        L.fjgen_rmat_device.restype = C.c_int
        L.fjgen_device_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _cache_dir():
    d = os.environ.get("FJG_DATA_CACHE", "/tmp/fjg_data")
    os.makedirs(d, exist_ok=True)
    return d


def _cached(key, fn, ncols):
    h = hashlib.sha1(repr(key).encode()).hexdigest()[:16]
    paths = [os.path.join(_cache_dir(), f"{key[0]}_{h}_{i}.npy") for i in range(ncols)]
    if all(os.path.exists(p) for p in paths):
        try:
            return [np.load(p) for p in paths]
        except Exception:
            pass
    cols = fn()
    for p, c in zip(paths, cols):
        tmp = p + f".tmp{os.getpid()}"
        np.save(tmp, c)
        os.replace(tmp + ".npy" if not tmp.endswith(".npy") else tmp, p)
    return cols


def uniform(seed, col, n, domain):
    out = np.empty(max(n, 1), dtype=np.int32)
    lib().fjgen_uniform(seed, col, n, domain, out.ctypes.data)
    return out[:n]


def zipf(seed, stream, n, k, s):
    def gen():
        out = np.empty(max(n, 1), dtype=np.int32)
        if lib().fjgen_zipf(seed, stream, n, k, s, out.ctypes.data) != 0:
            raise RuntimeError(lib().fjgen_last_error().decode())
        return [out[:n]]
    return _cached(("zipf", seed, stream, n, k, s), gen, 1)[0]


def rmat_device(seed, scale, m, a=0.57, b=0.19, c=0.19, device=0):
    """Same edges as rmat(), generated on the GPU into int32 CUDA tensors."""
    import torch
    src = torch.empty(max(m, 1), dtype=torch.int32, device=f"cuda:{device}")
    dst = torch.empty(max(m, 1), dtype=torch.int32, device=f"cuda:{device}")
    torch.cuda.synchronize(device)
    if lib().fjgen_rmat_device(device, seed, scale, m, a, b, c, src.data_ptr(), dst.data_ptr()) != 0:
        raise RuntimeError(lib().fjgen_device_last_error().decode())
    return src[:m], dst[:m]


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def rmat(seed, scale, m, a=0.57, b=0.19, c=0.19):
    """R-MAT edges: exactly m distinct directed non-loop edges, random row order.
    Large graphs are generated on the GPU when one is present (bit-identical)."""
    def gen():
        if m >= (1 << 26) and _gpu_available():
            s, d = rmat_device(seed, scale, m, a, b, c)
            return [s.cpu().numpy(), d.cpu().numpy()]
        s = np.empty(max(m, 1), dtype=np.int32)
        d = np.empty(max(m, 1), dtype=np.int32)
        if lib().fjgen_rmat(seed, scale, m, a, b, c, s.ctypes.data, d.ctypes.data) != 0:
            raise RuntimeError(lib().fjgen_last_error().decode())
        return [s[:m], d[:m]]
    return _cached(("rmat", seed, scale, m, a, b, c), gen, 2)


def orient(seed, src, dst):
    """Symmetrise, dedup, drop loops, orient by (degree, id)."""
    def gen():
        n = len(src)
        os_ = np.empty(max(n, 1), dtype=np.int32)
        od = np.empty(max(n, 1), dtype=np.int32)
        s = np.ascontiguousarray(src, dtype=np.int32)
        d = np.ascontiguousarray(dst, dtype=np.int32)
        k = lib().fjgen_orient(seed, s.ctypes.data, d.ctypes.data, n, os_.ctypes.data, od.ctypes.data)
        if k < 0:
            raise RuntimeError(lib().fjgen_last_error().decode())
        return [os_[:k].copy(), od[:k].copy()]
    key = ("orient", seed, len(src), hashlib.sha1(np.ascontiguousarray(src).tobytes()[:1 << 20]).hexdigest())
    return _cached(key, gen, 2)
