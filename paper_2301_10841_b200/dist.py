"""Multi-GPU Free Join: hash-partitioning on the first plan variable
(BASELINE.json north_star (c)).

One process per GPU (torch.distributed, NCCL over NVLink). Every rank starts
with a contiguous 1/G slice of each base relation (the distributed-load model).
Per step:
  1. views whose atom holds the plan's first variable v are hash-partitioned
     on v's column (fjg_relation_partition_into, fj::partition_of = fmix64 mod
     G) and exchanged with an all-to-all (uneven splits, counts exchanged
     first);
  2. every other view is all-gathered (padded to the largest slice, then
     compacted);
  3. each rank runs the single-GPU executor on (its shard of v) x (replicas);
     outputs are disjoint by v, so count = sum, checksum = sum mod 2^64,
     MIN = min, reduced with one all-reduce.
The exchange primitives take an `ops` object (array allocation + the
partition function) so the same exchange logic runs on CPU tensors under gloo
in tests/test_dist.py; the product path uses `DeviceOps` (the CUDA partition
kernel, NCCL).
"""
import torch
import torch.distributed as dist

MASK32 = (1 << 32) - 1


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


def _reuse(out, i, n, ops):
    """out[i] if it exists with n rows (persistent exchange buffers), else a new buffer."""
    if out is not None and i < len(out) and out[i].numel() == n:
        return out[i]
    return ops.empty(n)


def all_to_all_partitioned(grouped, counts, recv_counts, ops, group=None, out=None):
    """Rows already grouped by destination rank (partition_of(row[col]),
    `counts` per destination) -> this rank's rows, `recv_counts` per source
    (written into `out` when its buffers have the right sizes)."""
    res = []
    for i, g in enumerate(grouped):
        o = _reuse(out, i, sum(recv_counts), ops)
        dist.all_to_all_single(o, g, output_split_sizes=recv_counts, input_split_sizes=counts, group=group)
        res.append(o)
    return res


def all_gather_rows(cols, sizes, world, ops, group=None, out=None):
    """Every rank's rows of `cols` (`sizes` = each rank's row count),
    concatenated in rank order."""
    n = cols[0].numel() if cols else 0
    m = max(sizes) if sizes else 0
    res = []
    for i, c in enumerate(cols):
        if world == 1:
            o = _reuse(out, i, n, ops)
            o.copy_(c)
            res.append(o)
            continue
        pad = ops.empty(m)
        if n:
            pad[:n].copy_(c)
        buf = ops.empty(m * world)
        dist.all_gather_into_tensor(buf, pad, group=group)
        o = _reuse(out, i, sum(sizes), ops)
        off = 0
        for r in range(world):
            o[off: off + sizes[r]].copy_(buf[r * m: r * m + sizes[r]])
            off += sizes[r]
        res.append(o)
    return res


def reduce_results(count, checksum, minv, device, group=None):
    """count (python int, < 2^127), checksum (u64), minv (int or None) -> global.
    One all-gather of every rank's (count limbs, checksum halves, min) and a
    host-side sum / min: one collective and one device->host read per step."""
    INT64_MAX = (1 << 63) - 1
    parts = [count & MASK32, (count >> 32) & MASK32, (count >> 64) & MASK32, count >> 96,
             checksum & MASK32, checksum >> 32, INT64_MAX if minv is None else int(minv)]
    t = torch.tensor(parts, dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    if world == 1:
        rows = [t.tolist()]
    else:
        allp = torch.empty(world * len(parts), dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(allp, t, group=group)
        rows = allp.reshape(world, len(parts)).tolist()
    v = [sum(int(r[i]) for r in rows) for i in range(6)]
    total = v[0] + (v[1] << 32) + (v[2] << 64) + (v[3] << 96)
    cs = (v[4] + (v[5] << 32)) & ((1 << 64) - 1)
    mv = min(int(r[6]) for r in rows)
    return total, cs, (None if mv == INT64_MAX else mv)


def exchange(relations, views, world, rank, ops, group=None, bufs=None):
    """relations: base -> list of local-slice column tensors. Returns
    view -> list of column tensors held by this rank after the exchange
    (reusing `bufs`, the previous step's result, when sizes match).

    Every partitioned view is grouped by destination first; then ONE
    all-gather carries all size metadata (per partitioned view the counts
    per destination, per replicated view the local row count), so a step
    pays one metadata round trip however many views it exchanges."""
    order = sorted(set(views), key=lambda v: (v[0], -1 if v[1] is None else v[1]))
    meta, grouped = [], {}
    for view in order:
        base, col = view
        cols = relations[base]
        if col is None:
            meta.append([cols[0].numel() if cols else 0] * world)
        else:
            g, counts = ops.partition(cols, col, world)
            grouped[view] = (g, counts)
            meta.append(list(counts))
    nv = len(order)
    mine = torch.tensor(meta, dtype=torch.int64, device=ops.device).reshape(-1)
    if world == 1:
        allm = mine
    else:
        allm = torch.empty(world * nv * world, dtype=torch.int64, device=ops.device)
        dist.all_gather_into_tensor(allm, mine, group=group)
    M = allm.reshape(world, nv, world).tolist()  # M[source rank][view][destination]
    out = {}
    for vi, view in enumerate(order):
        base, col = view
        prev = bufs.get(view) if bufs else None
        if col is None:
            sizes = [int(M[r][vi][0]) for r in range(world)]
            out[view] = all_gather_rows(relations[base], sizes, world, ops, group, prev)
        else:
            g, counts = grouped[view]
            rc = [int(M[r][vi][rank]) for r in range(world)]
            out[view] = all_to_all_partitioned(g, counts, rc, ops, group, prev)
    return out


class DeviceOps:
    """Product ops: CUDA tensors, the libfjg partition kernel."""

    def __init__(self, engine):
        self.engine = engine
        self.device = torch.device("cuda", engine.device)
        self._send = {}  # (column pointers, key column) -> persistent send buffers

    def empty(self, n):
        return torch.empty(n, dtype=torch.int32, device=self.device)

    def partition(self, cols, col, world):
        key = (tuple(c.data_ptr() for c in cols), col)
        if key not in self._send:
            self._send[key] = (self.engine.relation_from_torch(cols), [self.empty(cols[0].numel()) for _ in cols])
        rel, grouped = self._send[key]
        counts = rel.partition_into(col, world, [g.data_ptr() for g in grouped])
        return grouped, counts


class ShardedQuery:
    """A workload executed across `world` ranks (one GPU each)."""

    def __init__(self, engine, w, plan, world, rank, group=None):
        from . import plan as P
        self.engine, self.w, self.plan = engine, w, plan
        self.world, self.rank, self.group = world, rank, group
        self.ops = DeviceOps(engine)
        self.fv, self.views = atom_views(w.query, w.atom_rel, plan)
        self.head = P.head_variables(w.query)
        # this rank's slice of every (filtered) base relation, resident on the device
        self.local = {}
        for base, cols in w.filtered().items():
            lo, hi = local_slice(len(cols[0]), world, rank)
            self.local[base] = [torch.from_numpy(c[lo:hi].copy()).to(self.ops.device) for c in cols]
        self.input_tuples_local = sum(len(w.relations[b][0]) for b in w.atom_rel) / world
        self._q = None
        self._eng_stream = torch.cuda.ExternalStream(engine.stream_ptr, device=self.ops.device)

    def _bind(self, held):
        rels = {v: self.engine.relation_from_torch(cols) for v, cols in held.items()}
        self._held = held
        self._rels = rels
        self._q = self.engine.query({"query": self.w.query}, self.plan, [rels[v] for v in self.views])

    def execute(self, min_var=None, timing=False, **kw):
        prev = getattr(self, "_held", None)
        held = exchange(self.local, self.views, self.world, self.rank, self.ops, self.group, prev)
        # the executor runs on the engine stream: order it after the exchange
        # on the device (no host synchronisation)
        self._eng_stream.wait_stream(torch.cuda.current_stream(self.ops.device))
        same = prev is not None and all(h is p for v in held for h, p in zip(held[v], prev[v]))
        # zero-copy relations over the exchanged buffers, bound once: every step
        # exchanges the same local slices, so the buffers' contents never change
        # under the bound query (relations are immutable; the query
        # caches per-relation facts such as a sorted root's key width)
        if self._q is None or not same:
            self._bind(held)
        r = self._q.execute(min_var=min_var, timing=timing, **kw)
        r.extra["local_count"] = r.count
        r.count, r.checksum, r.min_value = reduce_results(r.count, r.checksum, r.min_value, self.ops.device,
                                                          self.group)
        return r
