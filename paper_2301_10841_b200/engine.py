"""Device engine, relations and queries (host side of the C-ABI).

Mirrors the reference's trie/executor surface: relations are
immutable columnar tables; a Query binds a validated Free Join plan to one
relation per atom; Query.execute() runs the build phase (COLT `new`, lazy) and
the join phase (Fig 13 join_vectorized with dynamic cover) on the GPU and
returns the OutputSink counters plus ExecStats/TrieStats.
"""
import ctypes as C
import json
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check, lib

OUT_COUNT, OUT_ENUMERATE, OUT_FACTORIZED_COUNT = 0, 1, 2
_OUT = {"count": OUT_COUNT, "enumerate": OUT_ENUMERATE, "factorized_count": OUT_FACTORIZED_COUNT}
_BACKEND = {"colt": 0, "slt": 1, "simple": 2}  # FJG_BACKEND_*
CMP = {"=": 0, "==": 0, "!=": 1, "<": 2, "<=": 3, ">": 4, ">=": 5}


@dataclass
class ExecResult:
    count: int
    checksum: int
    min_value: object
    probes: int
    probe_misses: int
    node_body_entries: list
    node_probes: list
    node_inputs: list
    maps_built: int
    keys_inserted: int
    forces: int
    rows_forced: int
    build_ms: float
    join_ms: float
    last_node_ms: float
    last_node_launches: int
    last_node_candidates: int
    first_node_ms: float
    kernel_launches: int
    host_syncs: int
    output_rows: int = 0
    memo_ms: float = 0.0
    memo_rows: tuple = (0, 0, 0)  # resolved / gathered / initialised rows of the memo passes
    atom_maps_built: list = field(default_factory=list)     # TrieStats per atom (its physical trie)
    atom_levels_forced: list = field(default_factory=list)
    extra: dict = field(default_factory=dict)


class Engine:
    """One CUDA device + stream + memory pool (fjg_engine)."""

    def __init__(self, device=0):
        h = C.c_void_p()
        check(lib.fjg_engine_create(int(device), C.byref(h)))
        self._h = h
        self.device = device
        self._children = weakref.WeakSet()  # relations / queries: closed before the engine

    def close(self):
        if self._h:
            for c in list(self._children):
                c.close()
            lib.fjg_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(lib.fjg_engine_sync(self._h))

    @property
    def stream_ptr(self):
        """cudaStream_t the engine launches on (wrap with torch.cuda.ExternalStream)."""
        return lib.fjg_engine_stream(self._h)

    def relation(self, cols):
        """load columns (host int32 arrays) -> device Relation (fjg_relation_create)."""
        arrs = [np.ascontiguousarray(c, dtype=np.int32) for c in cols]
        n = len(arrs[0]) if arrs else 0
        if any(len(a) != n for a in arrs):
            raise _capi.ValidationError("all columns must have identical length (SPEC.md:35)")
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        h = C.c_void_p()
        check(lib.fjg_relation_create(self._h, ptrs, len(arrs), n, C.byref(h)))
        return Relation(self, h, keepalive=None)

    def relation_i64(self, cols):
        """load int64 host columns (fj::Value, value.hpp:31), narrowed on the device
        (fjg_relation_create_i64); ValidationError if a value does not fit int32."""
        arrs = [np.ascontiguousarray(c, dtype=np.int64) for c in cols]
        n = len(arrs[0]) if arrs else 0
        if any(len(a) != n for a in arrs):
            raise _capi.ValidationError("all columns must have identical length (SPEC.md:35)")
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        h = C.c_void_p()
        check(lib.fjg_relation_create_i64(self._h, ptrs, len(arrs), n, C.byref(h)))
        return Relation(self, h, keepalive=None)

    def relation_host_ptrs(self, ptrs, nrows):
        """fjg_relation_create from raw host column pointers (e.g. pinned buffers)."""
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        h = C.c_void_p()
        check(lib.fjg_relation_create(self._h, arr, len(ptrs), int(nrows), C.byref(h)))
        return Relation(self, h)

    def relation_from_device(self, ptrs, nrows, copy=False, keepalive=None):
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        h = C.c_void_p()
        check(lib.fjg_relation_from_device(self._h, arr, len(ptrs), int(nrows), int(bool(copy)), C.byref(h)))
        return Relation(self, h, keepalive=None if copy else keepalive)

    def relation_from_torch(self, tensors, copy=False):
        """Wrap CUDA int32 tensors (one per column) as a relation (zero-copy unless copy=True)."""
        for t in tensors:
            if not t.is_cuda or t.dtype.itemsize != 4 or not t.is_contiguous():
                raise _capi.ValidationError("columns must be contiguous CUDA int32 tensors")
        n = tensors[0].numel() if tensors else 0
        return self.relation_from_device([t.data_ptr() for t in tensors], n, copy=copy, keepalive=list(tensors))

    def query(self, query, plan, atom_relations):
        return Query(self, query, plan, atom_relations)

    def colt(self, relation, levels):
        """A GHT / COLT handle over `relation` (fjg_colt_create): `levels` = key
        column lists per level, e.g. [[0], [1]]."""
        return Colt(self, relation, levels)

    def device_tuple_hash(self, tuples):
        t = np.ascontiguousarray(np.asarray(tuples, dtype=np.int64))
        if t.ndim == 1:
            t = t.reshape(-1, 1) if t.size else t.reshape(0, 0)
        n, arity = (t.shape[0], t.shape[1]) if t.ndim == 2 else (0, 0)
        out = np.zeros(max(n, 1), dtype=np.uint64)
        check(lib.fjg_device_tuple_hash(self._h, t.ctypes.data, arity, n, out.ctypes.data))
        return out[:n]


class Relation:
    """Immutable device columnar relation."""

    def __init__(self, engine, handle, keepalive=None):
        self.engine = engine
        self._h = handle
        self._keep = keepalive
        engine._children.add(self)

    @property
    def rows(self):
        return int(lib.fjg_relation_rows(self._h))

    @property
    def ncols(self):
        return int(lib.fjg_relation_cols(self._h))

    def device_col(self, c):
        return lib.fjg_relation_device_col(self._h, c)

    def download(self):
        out = []
        for c in range(self.ncols):
            a = np.empty(max(self.rows, 1), dtype=np.int32)
            check(lib.fjg_relation_download(self._h, c, a.ctypes.data))
            out.append(a[: self.rows])
        return out

    def filter(self, preds):
        """apply_filter. preds: (col, op, const) or (col, op, ('col', c2))."""
        arr = (_capi.Predicate * max(len(preds), 1))()
        for i, (col, op, rhs) in enumerate(preds):
            arr[i].column = col
            arr[i].cmp = CMP[op]
            if isinstance(rhs, tuple):
                arr[i].is_column, arr[i].rhs_column = 1, rhs[1]
            else:
                arr[i].constant = int(rhs)
        h = C.c_void_p()
        check(lib.fjg_relation_filter(self._h, arr, len(preds), C.byref(h)))
        return Relation(self.engine, h)

    def partition(self, col, nparts):
        """Hash-partition rows on `col` (multi-GPU sharding): (relation grouped by part, counts)."""
        counts = (C.c_uint64 * nparts)()
        h = C.c_void_p()
        check(lib.fjg_relation_partition(self._h, col, nparts, C.byref(h), counts))
        return Relation(self.engine, h), [int(x) for x in counts]

    def partition_into(self, col, nparts, out_ptrs):
        """Hash-partition into caller-provided device columns; returns per-destination counts."""
        counts = (C.c_uint64 * nparts)()
        arr = (C.c_void_p * len(out_ptrs))(*out_ptrs)
        check(lib.fjg_relation_partition_into(self._h, col, nparts, arr, counts))
        return [int(x) for x in counts]

    def close(self):
        if self._h and self.engine._h:
            lib.fjg_relation_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Query:
    """A validated Free Join plan bound to one relation per query atom."""

    def __init__(self, engine, query, plan, atom_relations):
        self.engine = engine
        if isinstance(query, dict):
            qd = query
            head = query.get("head")
        elif isinstance(query, str):
            qd = json.loads(query)
            head = qd.get("head")
        else:
            qd = {"query": query}
            head = None
        self.atoms = qd["query"]
        self.query_json = json.dumps({"query": self.atoms, **({"head": head} if head else {})})
        self.plan = plan
        self.plan_json = plan if isinstance(plan, str) else json.dumps([[[r, list(v)] for (r, v) in n] for n in plan])
        self.relations = list(atom_relations)
        arr = (C.c_void_p * len(self.relations))(*[r._h.value for r in self.relations])
        h = C.c_void_p()
        check(lib.fjg_query_create(engine._h, self.query_json.encode(), self.plan_json.encode(), arr,
                                   len(self.relations), C.byref(h)))
        self._h = h
        engine._children.add(self)
        self.head = []
        for a in self.atoms:
            for v in a["vars"]:
                if v not in self.head:
                    self.head.append(v)
        if head:
            self.head = list(head)

    def execute(self, batch_size=0, dynamic_cover=True, output_mode="count", min_var=None, timing=False,
                backend="colt"):
        o = _capi.ExecOptions()
        o.backend = _BACKEND[backend] if isinstance(backend, str) else int(backend)
        o.batch_size = int(batch_size)
        o.dynamic_cover = int(bool(dynamic_cover))
        o.output_mode = _OUT[output_mode] if isinstance(output_mode, str) else int(output_mode)
        o.min_var = -1 if min_var is None else (self.head.index(min_var) if isinstance(min_var, str) else int(min_var))
        o.collect_timing = int(bool(timing))
        r = _capi.Result()
        check(lib.fjg_execute(self._h, C.byref(o), C.byref(r)))
        nn = r.num_nodes
        return ExecResult(count=(r.count_hi << 64) | r.count_lo, checksum=r.checksum,
                          min_value=(r.min_value if r.has_min else None), probes=r.probes,
                          probe_misses=r.probe_misses, node_body_entries=list(r.node_body_entries[:nn]),
                          node_probes=list(r.node_probes[:nn]), node_inputs=list(r.node_inputs[:nn]),
                          maps_built=r.maps_built, keys_inserted=r.keys_inserted, forces=r.forces,
                          rows_forced=r.rows_forced, build_ms=r.build_ms, join_ms=r.join_ms,
                          last_node_ms=r.last_node_ms, last_node_launches=r.last_node_launches,
                          last_node_candidates=r.last_node_candidates, first_node_ms=r.first_node_ms,
                          memo_ms=r.memo_ms, memo_rows=(r.memo_rows_resolved, r.memo_rows_gathered,
                                                        r.memo_rows_init),
                          atom_maps_built=list(r.atom_maps_built[:len(self.atoms)]),
                          atom_levels_forced=list(r.atom_levels_forced[:len(self.atoms)]),
                          kernel_launches=r.kernel_launches, host_syncs=r.host_syncs, output_rows=r.output_rows)

    def enumerate(self, batch_size=0, dynamic_cover=True, min_var=None, backend="colt"):
        """Enumerate mode: (tuples as an (n, |head|) int32 array in head-variable order, ExecResult)."""
        r = self.execute(batch_size=batch_size, dynamic_cover=dynamic_cover, output_mode="enumerate",
                         min_var=min_var, backend=backend)
        nv = len(self.head)
        buf = np.empty((max(r.output_rows, 1), nv), dtype=np.int32)
        rows = C.c_uint64(0)
        check(lib.fjg_query_output(self._h, buf.ctypes.data, r.output_rows, C.byref(rows)))
        return buf[: rows.value], r

    def output_relation(self):
        """After an enumerate execute: the output as a device Relation (one column per head var)."""
        h = C.c_void_p()
        check(lib.fjg_query_output_relation(self._h, C.byref(h)))
        return Relation(self.engine, h)

    def close(self):
        if self._h and self.engine._h:
            lib.fjg_query_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Colt:
    """Device GHT with the COLT interface of Fig 5 / Fig 12 (PAPER.md:544-557,
    SPEC.md:286-339): force / get / iter / rows / estimated_key_count over
    subtries named (p, len); state persists across calls."""

    def __init__(self, engine, relation, levels):
        flat = [int(c) for lv in levels for c in lv]
        cols = (C.c_int * max(len(flat), 1))(*flat)
        ncols = (C.c_int * len(levels))(*[len(lv) for lv in levels])
        h = C.c_void_p()
        check(lib.fjg_colt_create(engine._h, relation._h, cols, ncols, len(levels), C.byref(h)))
        self._h, self.engine, self.relation = h, engine, relation
        self.key_arity = [len(lv) for lv in levels]
        self.nlevels = lib.fjg_colt_levels(h)
        engine._children.add(self)

    def _arity(self, level):
        # out-of-range levels are reported by the library (ValidationError)
        return self.key_arity[level] if 0 <= level < len(self.key_arity) else 1

    def force(self, level, subtries):
        p = np.ascontiguousarray([s[0] for s in subtries], dtype=np.uint32)
        n = np.ascontiguousarray([s[1] for s in subtries], dtype=np.uint32)
        check(lib.fjg_colt_force(self._h, level, p.ctypes.data, n.ctypes.data, len(p)))

    def get(self, level, subtries, keys):
        """keys: one tuple per subtrie; returns [(child_p, child_len) or None]."""
        n = len(keys)
        ar = self._arity(level)
        p = np.ascontiguousarray([s[0] for s in subtries], dtype=np.uint32)
        ln = np.ascontiguousarray([s[1] for s in subtries], dtype=np.uint32)
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.int32).reshape(n, ar))
        cp = np.zeros(max(n, 1), dtype=np.uint32)
        cl = np.zeros(max(n, 1), dtype=np.uint32)
        f = np.zeros(max(n, 1), dtype=np.uint8)
        check(lib.fjg_colt_get(self._h, level, p.ctypes.data, ln.ctypes.data, k.ctypes.data, n, cp.ctypes.data,
                               cl.ctypes.data, f.ctypes.data))
        return [(int(cp[i]), int(cl[i])) if f[i] else None for i in range(n)]

    def iter(self, level, subtrie=(0, 0)):
        """Distinct keys of a map subtrie with their child subtries: [(key tuple, (p, len))]."""
        ar = self._arity(level)
        cap = max(int(subtrie[1]) if level else self.relation.rows, 1)
        keys = np.zeros(cap * ar, dtype=np.int32)
        cp = np.zeros(cap, dtype=np.uint32)
        cl = np.zeros(cap, dtype=np.uint32)
        n = C.c_uint64()
        check(lib.fjg_colt_iter(self._h, level, int(subtrie[0]), int(subtrie[1]), keys.ctypes.data, cp.ctypes.data,
                                cl.ctypes.data, cap, C.byref(n)))
        k = n.value
        return [(tuple(int(x) for x in keys[i * ar:(i + 1) * ar]), (int(cp[i]), int(cl[i]))) for i in range(k)]

    def rows(self, level, subtrie, col):
        out = np.zeros(max(int(subtrie[1]), 1), dtype=np.int32)
        check(lib.fjg_colt_rows(self._h, level, int(subtrie[0]), int(subtrie[1]), col, out.ctypes.data))
        return out[:int(subtrie[1])]

    def estimated_key_count(self, level, subtrie=(0, 0)):
        out = C.c_uint64()
        check(lib.fjg_colt_estimated_key_count(self._h, level, int(subtrie[0]), int(subtrie[1]), C.byref(out)))
        return out.value

    def close(self):
        if getattr(self, "_h", None):
            lib.fjg_colt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
