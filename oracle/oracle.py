"""ORACLE — TEST INFRASTRUCTURE ONLY. ctypes glue for oracle/liboracle.so, the
CPU restatement of the reference's Free Join path (oracle/fj_oracle.cpp)."""
import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

SIMPLE, SLT, COLT = 0, 1, 2
BACKENDS = {"simple": SIMPLE, "slt": SLT, "colt": COLT}


class OrcResult(C.Structure):
    _fields_ = [("count_lo", C.c_uint64), ("count_hi", C.c_uint64), ("checksum", C.c_uint64),
                ("min_value", C.c_int64), ("has_min", C.c_int32), ("factorized", C.c_int32),
                ("probes", C.c_uint64), ("probe_misses", C.c_uint64), ("node_body_entries", C.c_uint64 * 32),
                ("maps_built", C.c_uint64), ("keys_inserted", C.c_uint64), ("forces", C.c_uint64),
                ("atom_maps_built", C.c_uint64 * 16), ("atom_keys_inserted", C.c_uint64 * 16),
                ("atom_levels_forced", C.c_uint32 * 16)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2301_10841_b200/build.py")
        L = C.CDLL(LIB_PATH)
        P, I, U64 = C.c_void_p, C.c_int, C.c_uint64
        L.orc_execute.restype = I
        L.orc_execute.argtypes = [C.c_char_p, C.c_char_p, P, P, P, I, I, U64, I, I, I, I, I, I,
                                  C.POINTER(OrcResult), C.POINTER(P), C.POINTER(U64)]
        L.orc_brute_force.restype = I
        L.orc_brute_force.argtypes = [C.c_char_p, P, P, P, I, C.POINTER(P), C.POINTER(U64)]
        L.orc_free.argtypes = [P]
        L.orc_last_error.restype = C.c_char_p
        L.orc_tuple_hash.restype = U64
        L.orc_tuple_hash.argtypes = [P, I]
        L.orc_checksum_word.restype = U64
        L.orc_checksum_word.argtypes = [U64]
        L.orc_partition_of.restype = C.c_uint32
        L.orc_partition_of.argtypes = [C.c_int64, C.c_uint32]
        _lib = L
    return _lib


def _rel_args(atom_cols):
    """atom_cols: per atom, a list of int32 numpy columns."""
    keep = []
    col_ptr_arrays = []
    for cols in atom_cols:
        cs = [np.ascontiguousarray(c, dtype=np.int32) for c in cols]
        keep.extend(cs)
        col_ptr_arrays.append((C.c_void_p * len(cs))(*[c.ctypes.data for c in cs]))
    keep.extend(col_ptr_arrays)
    atom_ptrs = (C.c_void_p * len(atom_cols))(*[C.cast(a, C.c_void_p).value for a in col_ptr_arrays])
    ncols = (C.c_int * len(atom_cols))(*[len(c) for c in atom_cols])
    rows = (C.c_uint64 * len(atom_cols))(*[len(c[0]) if len(c) else 0 for c in atom_cols])
    keep.extend([atom_ptrs, ncols, rows])
    return atom_ptrs, ncols, rows, keep


def _qjson(query):
    if isinstance(query, str):
        return query
    if isinstance(query, dict):
        return json.dumps({"query": query["query"]})
    return json.dumps({"query": query})


def _pjson(plan):
    return plan if isinstance(plan, str) else json.dumps([[[r, list(v)] for (r, v) in n] for n in plan])


def execute(query, plan, atom_cols, backend="colt", batch_size=1000, dynamic_cover=True,
            output_mode="count", min_var=-1, part=0, nparts=1, nthreads=1):
    """Run the CPU oracle. Returns a dict (count, checksum, min, stats[, tuples])."""
    L = lib()
    atom_ptrs, ncols, rows, keep = _rel_args(atom_cols)
    om = {"count": 0, "enumerate": 1, "factorized_count": 2}[output_mode]
    res = OrcResult()
    tp = C.c_void_p()
    nt = C.c_uint64(0)
    rc = L.orc_execute(_qjson(query).encode(), _pjson(plan).encode(), atom_ptrs, ncols, rows, len(atom_cols),
                       BACKENDS[backend] if isinstance(backend, str) else backend, int(batch_size),
                       int(bool(dynamic_cover)), om, int(min_var), int(part), int(nparts), int(nthreads),
                       C.byref(res), C.byref(tp), C.byref(nt))
    if rc != 0:
        raise RuntimeError("oracle: " + L.orc_last_error().decode())
    out = {"count": (res.count_hi << 64) | res.count_lo, "checksum": res.checksum,
           "min": res.min_value if res.has_min else None, "factorized": bool(res.factorized),
           "probes": res.probes, "probe_misses": res.probe_misses,
           "node_body_entries": list(res.node_body_entries), "maps_built": res.maps_built,
           "keys_inserted": res.keys_inserted, "forces": res.forces,
           "atom_maps_built": list(res.atom_maps_built[:len(atom_cols)]),
           "atom_keys_inserted": list(res.atom_keys_inserted[:len(atom_cols)]),
           "atom_levels_forced": list(res.atom_levels_forced[:len(atom_cols)])}
    nv = len({v for a in json.loads(_qjson(query))["query"] for v in a["vars"]})
    if om == 1:
        arr = np.ctypeslib.as_array(C.cast(tp, C.POINTER(C.c_int64)), shape=(max(nt.value * nv, 1),))
        out["tuples"] = arr[: nt.value * nv].reshape(nt.value, nv).copy()
    L.orc_free(tp)
    del keep
    return out


def brute_force(query, atom_cols):
    """Nested-loop join bag, head-variable order."""
    L = lib()
    atom_ptrs, ncols, rows, keep = _rel_args(atom_cols)
    tp = C.c_void_p()
    nt = C.c_uint64(0)
    rc = L.orc_brute_force(_qjson(query).encode(), atom_ptrs, ncols, rows, len(atom_cols), C.byref(tp), C.byref(nt))
    if rc != 0:
        raise RuntimeError("oracle: " + L.orc_last_error().decode())
    nv = len({v for a in json.loads(_qjson(query))["query"] for v in a["vars"]})
    arr = np.ctypeslib.as_array(C.cast(tp, C.POINTER(C.c_int64)), shape=(max(nt.value * nv, 1),))
    out = arr[: nt.value * nv].reshape(nt.value, nv).copy()
    L.orc_free(tp)
    del keep
    return out


def tuple_hash(vals):
    a = np.ascontiguousarray(np.asarray(vals, dtype=np.int64))
    return int(lib().orc_tuple_hash(a.ctypes.data if a.size else None, len(a)))


def checksum_of(tuples):
    """sum fmix64(TupleHash(t)) mod 2^64 over a bag of tuples (rows)."""
    L = lib()
    s = 0
    for t in np.asarray(tuples, dtype=np.int64):
        s = (s + L.orc_checksum_word(tuple_hash(t))) & 0xFFFFFFFFFFFFFFFF
    return s


def partition_of(v, nparts):
    return int(lib().orc_partition_of(int(v), int(nparts)))
