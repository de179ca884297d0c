"""Multi-GPU Free Join: hash-partitioning on the first plan variable
(BASELINE.json north_star (c)), through the C-ABI (include/fjg.h
fjg_comm_* / fjg_sharded_* / fjg_execute_multi, csrc/multi.cuh).

One process per GPU. Every rank holds a contiguous 1/G slice of each base
relation (the distributed-load model). fjg_execute_multi then, on the engine
stream: hash-partitions the views holding the plan's first variable
(fj::partition_of = fmix64 mod G), all-gathers the size metadata once,
exchanges every view in one NCCL group (all-to-all of the partitioned views,
all-gather of the replicated ones), runs the single-GPU executor on the rows
it holds, and all-reduces (count, checksum, MIN): outputs are disjoint by the
first variable. torch.distributed is used here only to ship the 128-byte NCCL
id from rank 0 to the other ranks (any channel would do).
"""
import ctypes as C
import json

import numpy as np

from . import _capi
from ._capi import check, lib
from .engine import ExecResult, _OUT, _BACKEND


def first_variable(plan):
    node0 = plan[0]
    for (_, vs) in node0:
        if vs:
            return vs[0]
    raise ValueError("plan binds no variable in its first node")


def atom_views(query, atom_rel, plan):
    """Per atom: (base relation, column of the first variable or None)."""
    fv = first_variable(plan)
    views = []
    for atom, base in zip(query, atom_rel):
        views.append((base, atom["vars"].index(fv) if fv in atom["vars"] else None))
    return fv, views


def local_slice(n, world, rank):
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi


class Comm:
    """fjg_comm: one NCCL communicator per rank on the engine's device."""

    def __init__(self, engine, world, rank, uid=None, group=None):
        if uid is None:
            buf = C.create_string_buffer(_capi.COMM_ID_BYTES)
            if rank == 0:
                check(lib.fjg_comm_unique_id(buf))
            if world > 1:
                import torch.distributed as dist
                obj = [bytes(buf.raw) if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                buf = C.create_string_buffer(obj[0], _capi.COMM_ID_BYTES)
            uid = buf
        h = C.c_void_p()
        check(lib.fjg_comm_create(engine._h, uid, int(world), int(rank), C.byref(h)))
        self._h, self.engine, self.world, self.rank = h, engine, world, rank

    def close(self):
        if self._h:
            lib.fjg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedQuery:
    """A workload executed across the ranks of `comm` (one GPU each)."""

    def __init__(self, engine, w, plan, comm, local=None):
        """local: optional base -> this rank's columns (numpy arrays, or host
        torch tensors copied from their pointers); default: slice w's relations."""
        from . import plan as P
        self.engine, self.w, self.plan, self.comm = engine, w, plan, comm
        world, rank = comm.world, comm.rank
        self.fv, self.views = atom_views(w.query, w.atom_rel, plan)
        self.head = P.head_variables(w.query)
        bases = sorted(set(w.atom_rel))
        # this rank's slice of every (filtered) base relation, resident on the device
        self.local = {}
        self._rels = {}
        for base in bases:
            cols = (local or {}).get(base)
            if cols is None:
                full = w.filtered()[base]
                lo, hi = local_slice(len(full[0]), world, rank)
                cols = [np.ascontiguousarray(c[lo:hi]) for c in full]
            if hasattr(cols[0], "data_ptr"):  # host tensors (e.g. pinned): H2D from their pointers
                self._rels[base] = engine.relation_host_ptrs([c.data_ptr() for c in cols], cols[0].numel())
            else:
                self._rels[base] = engine.relation(cols)
            self.local[base] = cols
        self.input_tuples_local = sum(len(w.relations[b][0]) for b in w.atom_rel) / world
        arr = (C.c_void_p * len(bases))(*[self._rels[b]._h.value for b in bases])
        ab = (C.c_int * len(w.atom_rel))(*[bases.index(b) for b in w.atom_rel])
        fc = (C.c_int * len(w.atom_rel))(*[-1 if c is None else c for (_, c) in self.views])
        h = C.c_void_p()
        check(lib.fjg_sharded_create(comm._h, json.dumps({"query": w.query}).encode(),
                                     json.dumps([[[r, list(v)] for (r, v) in n] for n in plan]).encode(),
                                     arr, len(bases), ab, fc, len(w.atom_rel), C.byref(h)))
        self._h = h

    def execute(self, min_var=None, timing=False, batch_size=0, dynamic_cover=True, output_mode="count",
                backend="colt"):
        o = _capi.ExecOptions()
        o.batch_size = int(batch_size)
        o.dynamic_cover = int(bool(dynamic_cover))
        o.output_mode = _OUT[output_mode]
        o.min_var = self.head.index(min_var) if isinstance(min_var, str) else (-1 if min_var is None else min_var)
        o.collect_timing = int(bool(timing))
        o.backend = _BACKEND[backend]
        r = _capi.Result()
        info = _capi.MultiInfo()
        check(lib.fjg_execute_multi(self._h, C.byref(o), C.byref(r), C.byref(info)))
        n = r.num_nodes
        res = ExecResult(
            count=(r.count_hi << 64) | r.count_lo, checksum=r.checksum,
            min_value=r.min_value if r.has_min else None, probes=r.probes, probe_misses=r.probe_misses,
            node_body_entries=list(r.node_body_entries[:n]), node_probes=list(r.node_probes[:n]),
            node_inputs=list(r.node_inputs[:n]), maps_built=r.maps_built, keys_inserted=r.keys_inserted,
            forces=r.forces, rows_forced=r.rows_forced, build_ms=r.build_ms, join_ms=r.join_ms,
            last_node_ms=r.last_node_ms, last_node_launches=r.last_node_launches,
            last_node_candidates=r.last_node_candidates, first_node_ms=r.first_node_ms,
            memo_ms=r.memo_ms, memo_rows=(r.memo_rows_resolved, r.memo_rows_gathered, r.memo_rows_init),
            kernel_launches=r.kernel_launches, host_syncs=r.host_syncs, output_rows=r.output_rows)
        res.extra["local_count"] = (info.local_count_hi << 64) | info.local_count_lo
        res.extra["local_checksum"] = info.local_checksum
        res.extra["bytes_sent"] = info.bytes_sent
        res.extra["bytes_received"] = info.bytes_received
        res.extra["view_rows"] = list(info.view_rows[:info.nviews])
        res.extra["exchange_ms"] = info.exchange_ms
        res.extra["reduce_ms"] = info.reduce_ms
        return res

    def close(self):
        if getattr(self, "_h", None):
            lib.fjg_sharded_destroy(self._h)
            self._h = None
        for r in self._rels.values():
            r.close()
        self._rels = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
