"""Per-rank executor time at G ranks, measured on ONE GPU without NCCL: the
full relations are partitioned on the plan's first variable with the product
partition kernel (fjg_relation_partition_into; a stable partition of the whole
relation holds exactly the rows, in the same order, that rank r receives from
the all-to-all over contiguous slices), the other views are the full
relations (the replicas), and each rank's query is timed alone (CUDA events,
L2 flushed between steps). The sum of the G ranks' counts / checksums must
equal the single-GPU result. Exchange and result reduction are NOT included
(they need G GPUs). Usage: python scripts/rank_shard_estimate.py [config] [G ...]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs, dist as D
from paper_2301_10841_b200 import plan as P

name = sys.argv[1] if len(sys.argv) > 1 else "triangle"
Gs = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
eng = fjg.Engine(0)
stream = torch.cuda.ExternalStream(eng.stream_ptr, device=torch.device("cuda", 0))
flush = torch.empty(2 * 126 * (1 << 20) // 4, dtype=torch.int32, device="cuda")
w = configs.CONFIGS[name]()
plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
fv, views = D.atom_views(w.query, w.atom_rel, plan)
full = {b: [torch.from_numpy(c).cuda() for c in cols] for b, cols in w.filtered().items()}


def partition(cols, col, G):
    """The product partition kernel (fjg_relation_partition_into) into torch buffers."""
    rel = eng.relation_from_torch(cols)
    grouped = [torch.empty_like(c) for c in cols]
    counts = rel.partition_into(col, G, [g.data_ptr() for g in grouped])
    rel.close()
    return grouped, counts


BIG = name.startswith("scale")


def timed(q, steps=2 if BIG else 5):
    for _ in range(1 if BIG else 3):
        r = q.execute(min_var=w.min_var, output_mode=w.output_mode)
    ms = []
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = q.execute(min_var=w.min_var, output_mode=w.output_mode)
        e1.record(stream)
        eng.sync()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms), r


base_ms = None
for G in Gs:
    parts = {}
    for (b, col) in set(views):
        if col is None:
            continue
        grouped, counts = partition(full[b], col, G)
        offs = [sum(counts[:r]) for r in range(G)]
        parts[(b, col)] = [[g[offs[r]: offs[r] + counts[r]].clone() for g in grouped] for r in range(G)]
    total, cs, per = 0, 0, []
    for r in range(G):
        held = {v: (full[v[0]] if v[1] is None else parts[v][r]) for v in set(views)}
        rels = {v: eng.relation_from_torch(cols) for v, cols in held.items()}
        q = eng.query({"query": w.query}, plan, [rels[v] for v in views])
        ms, res = timed(q)
        total += res.count
        cs = (cs + res.checksum) & ((1 << 64) - 1)
        per.append(ms)
        q.close()
        for x in rels.values():
            x.close()
    mx = max(per)
    if base_ms is None and G == 1:
        base_ms = mx
    eff = (base_ms / (G * mx)) if base_ms else float("nan")
    print(f"{name} G={G}: per-rank query ms max {mx:.3f} mean {statistics.mean(per):.3f} "
          f"(efficiency excluding exchange vs G=1 sharded: {eff:.2f}) count {total} checksum {cs:#018x}", flush=True)
