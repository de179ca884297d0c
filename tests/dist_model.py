"""CPU model of the multi-GPU exchange protocol of fjg_execute_multi
(paper_2301_10841_b200/csrc/multi.cuh), written over torch.distributed so it
runs under gloo at world size > 1 without GPUs (tests/test_dist.py). Same
steps: partition the first-variable views, ONE all-gather of the size
metadata M[src][view][dst], all-to-all of partitioned views and all-gather of
replicated ones into rank order, per-rank execution, reduction of (count as
32-bit limbs, checksum halves, MIN). The C++ receive layout
(fjg_exchange_layout) is checked against `recv_layout` below. Test
infrastructure."""
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


def recv_layout(M, view_partitioned, rank):
    """Receive offsets per view and source rank, as fjg_execute_multi lays them out."""
    world = len(M)
    offs, rows = [], []
    for v, part in enumerate(view_partitioned):
        o = [0]
        for src in range(world):
            o.append(o[-1] + (M[src][v][rank] if part else M[src][v][0]))
        offs.append(o[:-1])
        rows.append(o[-1])
    return offs, rows
