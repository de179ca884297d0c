#!/usr/bin/env python
"""Benchmark: Free Join query throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config scale_triangle] [--impl ours|reference]

Default workload: C5 triangle (BASELINE configs[4]: R-MAT 2^27 vertices, 512M
edges), the config BASELINE.json's 1/2/4/8-GPU metric is quoted on.

A step = one full query execution (COLT build phase + join phase)
over inputs already resident in HBM. `value` = (input tuples + output tuples)
per second over the whole job; `e2e` = the same metric through the public
C-ABI with host (pinned) input buffers copied inside the timed region.
For N>1 (torchrun), relations holding the first plan variable are
hash-partitioned across ranks by an NCCL all-to-all and the rest all-gathered
(paper_2301_10841_b200/dist.py); the exchange is inside the timed step.
--impl reference times the CPU restatement of the reference path (oracle/)
over a bounded sample of the same workload; it loads only oracle/ libraries
(inputs from oracle/gen.cpp, plans from oracle/workload_plans.json).
--gpus N without torchrun re-launches this script under torch.distributed.run
with N ranks on 127.0.0.1.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "join tuples/sec (input+output) per query"
UNIT = "tuples/s"
L2_BYTES = 126 * (1 << 20)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="scale_triangle")
    ap.add_argument("--small", action="store_true", help="tiny sizes of the config (launcher / harness tests)")
    ap.add_argument("--cpu-threads", type=int, default=0, help="all-core CPU leg threads (0: every host thread)")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-target-s", type=float, default=20.0)
    ap.add_argument("--backend", default="colt", choices=["colt", "slt", "simple"],
                    help="GHT backend (SPEC.md:286-294): the §5.3 ablation ladder")
    ap.add_argument("--shard", action="store_true",
                    help="use the multi-GPU sharded path (partition + NCCL exchange) even at one rank")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


SMALL = {"chain": dict(n=20000, domain=30000), "triangle": dict(scale=12, m=30000),
         "star": dict(nf=50000, dims=(500, 400, 300, 200)), "clique4": dict(scale=12, m=30000),
         "path5": dict(scale=10, m=8000), "scale_triangle": dict(scale=14, m=100000),
         "scale_path5": dict(scale=14, m=100000)}


def workload(name, small=False):
    from paper_2301_10841_b200 import configs
    return configs.CONFIGS[name](**(SMALL[name] if small else {}))


def oracle_workload(name, small=False):
    """The same config restated on the oracle side (no product library)."""
    from oracle import workloads as OW
    return OW.CONFIGS[name](**(SMALL[name] if small else {}))


def config_dict(name, params, mode, backend):
    """Identical in both arms (the driver compares them)."""
    return {"workload": name, **params, "plan_mode": mode, "backend": backend}


def host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable"):
                    mem = int(line.split()[1]) * 1024
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "mem_available_bytes": mem}


def maybe_relaunch(args):
    """--gpus N outside torchrun: re-exec under torch.distributed.run, N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


class Clocks:
    """nvidia-smi sampler DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def node_entry_bytes(plan, query, k):
    """Bytes of one frontier entry entering node k (SoA: bound vars int32,
    open-atom subtrie (id,len) 2x u32, multiplicity u64) + chosen u8 + scan u64."""
    atoms = {a["rel"]: a for a in query}
    bound = set()
    for j in range(k):
        for (_, vs) in plan[j]:
            bound.update(vs)
    open_atoms = 0
    for name in atoms:
        nodes = [j for j, node in enumerate(plan) for (r, _) in node if r == name]
        if nodes and min(nodes) < k <= max(nodes):
            open_atoms += 1
    return 4 * len(bound) + 8 * open_atoms + (8 if k > 0 else 0) + 1 + 8


def last_node_bytes(plan, query, res):
    """SURVEY.md §8(d) sector model for the fused last-node kernel of one launch:
    32 B per probe (one sector per get) + the contiguous streams: frontier
    entries, cover values (int32 per candidate per cover variable)."""
    k = len(plan) - 1
    F = res.node_inputs[k]
    M = res.last_node_candidates
    P = res.node_probes[k]
    nv = max(len(vs) for (_, vs) in plan[k])
    seq = F * node_entry_bytes(plan, query, k) + M * 4 * nv
    return 32 * P + 32 * ((seq + 31) // 32)


def first_node_bytes(plan, query, res):
    """Sector model for node 0 of a stream plan (C1 / C3): the cover rows'
    first-probe key column streamed (4 B per row), 32 B per probe, one sector
    per later-probe key gathered for a row still alive, and the survivors'
    frontier entries written."""
    n = res.node_body_entries[0]
    P = res.node_probes[0]
    seq = 4 * n + (res.node_inputs[1] * node_entry_bytes(plan, query, 1) if len(plan) > 1 else 0)
    return 32 * P + 32 * max(P - n, 0) + 32 * ((seq + 31) // 32)


def memo_bytes(res):
    """Sector model of the memoised chain passes (factorised count): a resolved
    row streams its carrier value (4 B), probes one root (32 B) and writes its
    child (4 B); a gathered row streams gid + child (8 B) and gathers one memo
    entry (one 32 B sector); an initialising row streams cnt + gid (8 B)."""
    rr, rg, ri = res.memo_rows
    return 40 * rr + 40 * rg + 8 * ri


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.shard:
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------- CPU leg ---
# The CPU restatement of the reference path (oracle/fj_oracle.cpp) on the
# host cores. A sample = T threads, thread t running first-variable hash
# partition t of P with its own trie set (one independent trie
# instance per concurrent execution). The rows of the atoms that hold the
# first variable are restricted to the sampled partitions before the timed
# call (the host-side counterpart of the multi-GPU exchange; otherwise every
# thread would force those atoms' whole roots); atoms without it are whole.
# P starts large and shrinks 4x while the sample stays short, so a sample is
# bounded by ~target_s unless one thread's fixed trie build alone exceeds it.

def _np_partition_of(v, nparts):
    """fj::partition_of (csrc/fj_hash.hpp): fmix64(v ^ 0x5bd1e995) mod nparts."""
    import numpy as np
    with np.errstate(over="ignore"):
        k = v.astype(np.int64).astype(np.uint64) ^ np.uint64(0x5bd1e995)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xff51afd7ed558ccd)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xc4ceb9fe1a85ec53)
        k ^= k >> np.uint64(33)
    return k % np.uint64(nparts)


def _first_var_atoms(ow):
    plan = ow.plan
    fv = plan[0][0][1][0]
    return fv, [i for i, a in enumerate(ow.query) if fv in a["vars"]]


_PART_CACHE = {}


def _restricted_columns(ow, cols, T, P):
    """The atoms holding the first variable, restricted to partitions 0..T-1 of P
    (partition ids cached per (column, P): the C5 columns have 512M rows)."""
    fv, atoms = _first_var_atoms(ow)
    out = list(cols)
    for i in atoms:
        c = ow.query[i]["vars"].index(fv)
        key = (id(cols[i][c]), P)
        if key not in _PART_CACHE:
            _PART_CACHE.clear()
            _PART_CACHE[key] = _np_partition_of(cols[i][c], P)
        keep = _PART_CACHE[key] < T
        out[i] = [x[keep] for x in cols[i]]
    return out


def _thread_bytes(ow, cols, frac):
    """Per-thread trie footprint of the oracle (bytes): measured ~64 B per row of
    every whole atom (C5: 33 GB for the 512M-row E2 trie, one thread, maxrss
    41.7 GB with the inputs), the restricted atoms scaled by the fraction."""
    _, atoms = _first_var_atoms(ow)
    rows = sum(len(c[0]) * (frac if i in atoms else 1.0) for i, c in enumerate(cols))
    return int(64 * rows) + (256 << 20)


def cpu_sample(ow, T, P, cols=None):
    """One timed oracle sample: T threads, partitions 0..T-1 of P."""
    from oracle import oracle
    cols = cols if cols is not None else ow.atom_columns()
    head = ow.head()
    mv = head.index(ow.min_var) if ow.min_var else -1
    rc = _restricted_columns(ow, cols, T, P) if P > T else cols
    t0 = time.perf_counter()
    r = oracle.execute(ow.query, ow.plan, rc, part=0, nparts=P, nthreads=T, min_var=mv,
                       output_mode=ow.output_mode)
    dt = time.perf_counter() - t0
    frac = T / P
    units = ow.input_tuples() * frac + (r["count"] if ow.output_mode == "count" else 0)
    return {"value": units / dt, "seconds": dt, "threads": T, "P": P, "frac": frac, "count": r["count"],
            "checksum": r["checksum"], "min": r["min"]}


def cpu_leg(ow, T, target_s, cols=None):
    """Adaptive bounded sample on T threads: P starts at 4096 first-variable
    partitions and shrinks 4x while a sample takes < target_s/5, so the final
    sample is ~target_s unless one thread's fixed trie build alone is longer
    (C5: ~150 s to build the 512M-row E2 trie on one core)."""
    cols = cols if cols is not None else ow.atom_columns()
    # every thread starts with 1/4096 of the query: when a sample is dominated by
    # one thread's fixed trie build, T threads then do T times the work in the
    # same time (P = 4096 for every T), as they would on the whole query
    P = max(4096, T)
    s = cpu_sample(ow, T, P, cols)
    while P > T and s["seconds"] < target_s / 5:
        P = max(T, P // 4)
        s = cpu_sample(ow, T, P, cols)
    what = "the whole query" if P == T else f"{T} of {P} first-variable hash partitions ({s['frac']:.6f} of the query)"
    s["sample"] = (f"{what}; {T} thread(s), one independent trie set each (SPEC.md:354); rows of the first-variable"
                   f" atoms restricted to the sampled partitions before timing; input tuples scaled by the fraction")
    return s


def cpu_baseline(ow, target_s, threads=0, cols=None):
    """Single-thread (the reference's concurrency model) and
    all-core figures. The all-core thread count is capped by host memory (each
    thread holds its own tries)."""
    info = host_info()
    cols = cols if cols is not None else ow.atom_columns()
    one = cpu_leg(ow, 1, target_s, cols)
    T = threads or max(1, min(os.cpu_count() or 1, 64))
    capped = ""
    if info["mem_available_bytes"]:
        per = _thread_bytes(ow, cols, 1.0 / max(T, 1))
        tmax = max(1, int(0.75 * info["mem_available_bytes"] // per))
        if tmax < T:
            T, capped = tmax, f" (capped from {os.cpu_count()} by host memory: ~{per / 2**30:.1f} GiB of tries per thread)"
    allc = cpu_leg(ow, T, target_s, cols) if T > 1 else one
    keep = ("value", "seconds", "threads", "P", "frac", "sample")
    return {"value": allc["value"], "unit": UNIT, "cores": allc["threads"], "kind": "port",
            "sample": allc["sample"] + capped,
            "single_thread": {k: one[k] for k in keep},
            "all_core": {k: allc[k] for k in keep},
            "nproc": info["nproc"], "cpu_model": info["cpu_model"],
            "compiler": "g++ -O3 -march=x86-64-v2, batch 1000, dynamic cover (SPEC.md:502)"}


def run_reference(args):
    """The reference arm: oracle only (inputs oracle/gen.cpp, plan
    oracle/workload_plans.json); rank 0 runs, other ranks exit."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ow = oracle_workload(args.config, args.small)
    cols = ow.atom_columns()
    T = args.cpu_threads or max(1, min(os.cpu_count() or 1, 64))
    info = host_info()
    if info["mem_available_bytes"]:
        T = max(1, min(T, int(0.75 * info["mem_available_bytes"] // _thread_bytes(ow, cols, 1.0 / T))))
    steps = max(args.steps, 1)
    budget = 300.0  # seconds for the whole arm
    target = max(2.0, min(60.0, budget / (steps + args.warmup + 2)))
    s0 = cpu_leg(ow, T, target, cols)  # fixes P for every step (and warms the host caches)
    # a sample cannot be shorter than one thread's trie build: when K + W samples
    # of that size exceed the budget, run as many as fit (at least one)
    warm = args.warmup if s0["seconds"] * (steps + args.warmup) <= budget else 0
    steps = steps if s0["seconds"] * (steps + warm) <= budget else max(1, int(budget // max(s0["seconds"], 1e-9)))
    if steps == 1 and warm == 0 and s0["seconds"] > budget / 2:
        runs = [s0]  # the calibration sample already is one full-size step (same P, same threads)
    else:
        for _ in range(warm):
            cpu_sample(ow, T, s0["P"], cols)
        runs = [cpu_sample(ow, T, s0["P"], cols) for _ in range(steps)]
    v = statistics.median(r["value"] for r in runs)
    last = runs[-1]
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": 1000 * statistics.median(r["seconds"] for r in runs),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded generators)",
            "config": config_dict(ow.name, ow.params, ow.mode, args.backend),
            "impl": "reference",
            "parallelism": f"cpu-threads x{T}",
            "result": {"count": last["count"], "checksum": f"{last['checksum']:#018x}",
                       "min": last["min"], "output_mode": ow.output_mode,
                       "scope": "whole query" if last["P"] == T else f"partitions 0..{T - 1} of {last['P']}"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": T, "kind": "port", "sample": s0["sample"],
                             "nproc": info["nproc"], "cpu_model": info["cpu_model"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg ---
def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = dist_setup(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    import paper_2301_10841_b200 as fjg
    from paper_2301_10841_b200 import plan as P

    w = workload(args.config, args.small)
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    head = P.head_variables(w.query)
    mv = w.min_var
    eng = fjg.Engine(local)
    stream = torch.cuda.ExternalStream(eng.stream_ptr, device=torch.device("cuda", local))
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")

    if world > 1 or args.shard:
        from paper_2301_10841_b200 import dist as D
        comm = D.Comm(eng, world, rank)  # fjg_comm: NCCL, bootstrapped over torch.distributed
        sharded = D.ShardedQuery(eng, w, plan, comm)
        step = lambda timing=False: sharded.execute(min_var=mv, timing=timing, batch_size=args.batch,  # noqa: E731
                                                    output_mode=w.output_mode, backend=args.backend)
        input_tuples_local = sharded.input_tuples_local
    else:
        q, _, rels = fjg.prepare_workload(eng, w)
        step = lambda timing=False: q.execute(min_var=mv, timing=timing, batch_size=args.batch,  # noqa: E731
                                              output_mode=w.output_mode, backend=args.backend)
        input_tuples_local = w.input_tuples()

    for _ in range(max(args.warmup, 1)):
        res = step()
    # ---- timed region: K steps, device events on the engine stream ----
    clocks = Clocks(local)
    barrier(world)
    torch.cuda.synchronize()
    eng.sync()
    clocks.start()
    t_wall0 = time.perf_counter()
    evs = []
    results = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step(timing=True)
        e1.record(stream)
        with torch.cuda.stream(stream):
            flush.add_(1)  # L2 flush between timed steps (outside the event pair)
        evs.append((e0, e1))
        results.append(res)
    eng.sync()
    torch.cuda.synchronize()
    barrier(world)
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for (a, b) in evs]
    dev_ms_total = sum(step_ms)
    dev_ms_total = allreduce_max(dev_ms_total, world)
    ms_per_step = dev_ms_total / args.steps
    out_local = results[-1].extra.get("local_count", results[-1].count)
    # the 5-path count (~5e21) is computed factorised, not enumerated: count input tuples only
    units_local = input_tuples_local + (out_local if w.output_mode == "count" else 0)
    units = allreduce_sum(units_local, world)
    value = units / (ms_per_step / 1000.0)
    launches = sum(r.kernel_launches for r in results)

    # ---- roofline: the dominant node kernel (see profiles/) ----
    # the fused last node, or node 0 when it takes longer (the stream node of
    # C1 / C3: every fact row read and probed there, a few survivors after)
    hbm, hbm_kind = peaks()
    r0 = results[-1]
    last_ms = statistics.mean(r.last_node_ms / max(r.last_node_launches, 1) for r in results)
    last_bytes = last_node_bytes(plan, w.query, r0) / max(r0.last_node_launches, 1)
    first_ms = statistics.mean(r.first_node_ms for r in results)
    kernel = "fused last node (k_last_gj_warp for GJ-shaped nodes, k_tail for a Cartesian tail, else k_expand<COUNT>)"
    memo_ms = statistics.mean(r.memo_ms for r in results)
    cands = [(statistics.mean(r.last_node_ms for r in results), "last")]
    if world == 1:
        cands.append((first_ms, "first"))
    cands.append((memo_ms, "memo"))
    dom = max(cands)[1]
    if dom == "first":
        last_ms, last_bytes = first_ms, first_node_bytes(plan, w.query, r0)
        kernel = "node 0 (k_stream_one: single-binding stream node)"
    elif dom == "memo":
        last_ms, last_bytes = memo_ms, memo_bytes(r0)
        kernel = "memoised chain passes (k_memo_init / k_memo_resolve / k_memo_gather), one phase"
    achieved = last_bytes / (last_ms / 1000.0) / 1e9 if last_ms > 0 else 0.0
    # DRAM bytes per launch of the same kernel on the same workload, from this
    # round's committed ncu capture (profiles/r02_traffic_<workload>.json)
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"r02_traffic_{w.name}.json")
    if os.path.exists(tp) and world == 1 and dom == "last":
        with open(tp) as f:
            tj = json.load(f)
        # per launch of THIS run: the capture's DRAM bytes per execution over the run's launch count
        traffic = (tj["dram_bytes_per_execution"] / max(r0.last_node_launches, 1)
                   if "dram_bytes_per_execution" in tj else tj.get("dram_bytes_per_launch"))

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        if world > 1 or args.shard:
            e2e = e2e_leg_sharded(sharded, w, mv, args.e2e_steps, flush, world, args.backend)
        else:
            # return the warm query's tries and relations to the pool first, so the
            # e2e leg's query reuses that memory instead of holding a second trie set
            q.close()
            for r in rels.values():
                r.close()
            e2e = e2e_leg(fjg, eng, w, stream, mv, args.e2e_steps, flush)

    # ---- CPU baseline (rank 0, N=1): the oracle on the same bytes ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import workloads as OW
            ow = OW.OWorkload(w.name, w.query, w.atom_rel, w.relations, filters=w.filters, min_var=w.min_var,
                              params=w.params, output_mode=w.output_mode, mode=w.mode,
                              plan_override=[[[r, list(vs)] for (r, vs) in node] for node in plan])
            cpu = cpu_baseline(ow, args.cpu_target_s, args.cpu_threads)
        except Exception as ex:  # the CPU leg must not sink the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic (seeded generators, resident in HBM)",
            "config": config_dict(w.name, w.params, w.mode, args.backend),
            "parallelism": f"hash-partition x{world}" if (world > 1 or args.shard) else "single-gpu",
            "l2": "flushed between timed steps (2x126MB write)",
            "tuples": {"input": w.input_tuples(), "output": res.count if w.output_mode == "count" else 0},
            "result": {"count": res.count, "checksum": f"{res.checksum:#018x}", "min": res.min_value,
                       "output_mode": w.output_mode, "scope": "whole query"},
            "phases_ms": {"build": statistics.mean(r.build_ms for r in results),
                          "join": statistics.mean(r.join_ms for r in results),
                          "last_node_total": statistics.mean(r.last_node_ms for r in results),
                          "first_node": first_ms, "memo": memo_ms,
                          "last_node_per_launch": last_ms, "last_node_launches": r0.last_node_launches},
            "counters": {"probes": r0.probes, "node_probes": r0.node_probes, "node_inputs": r0.node_inputs,
                         "last_node_candidates": r0.last_node_candidates, "maps_built": r0.maps_built,
                         "keys_inserted": r0.keys_inserted, "host_syncs": r0.host_syncs},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "kernel": kernel,
                         "algorithmic_bytes_per_launch": last_bytes, "peak_kind": hbm_kind},
            "gpu_launches": launches,
            "clocks": clk,
            "wall_s": t_wall,
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1 or args.shard:
        import torch.distributed as dist
        dist.destroy_process_group()


def e2e_leg(fjg, eng, w, stream, mv, steps, flush):
    """Public API end to end: pinned host columns -> fjg_relation_create (H2D)
    -> filter -> plan compile -> fjg_query_create -> fjg_execute -> result D2H."""
    import torch
    host = {name: [torch.from_numpy(c).pin_memory() for c in cols] for name, cols in w.relations.items()}
    h2d = sum(t.numel() * 4 for cols in host.values() for t in cols)
    d2h = 8 * 160  # result counters block (fjg_result / DevCounters) per step
    times = []
    units = None
    for i in range(steps + 1):
        eng.sync()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        rels = {}
        for name, cols in host.items():
            r = eng.relation_host_ptrs([c.data_ptr() for c in cols], cols[0].numel())
            if w.filters.get(name):
                r = r.filter(w.filters[name])
            rels[name] = r
        q, _, _ = fjg.prepare_workload(eng, w, device_relations=rels)
        res = q.execute(min_var=mv, output_mode=w.output_mode)
        e1.record(stream)
        eng.sync()
        wall = time.perf_counter() - t0
        q.close()
        for r in rels.values():
            r.close()
        with torch.cuda.stream(stream):
            flush.add_(1)
        if i > 0:  # first iteration warms the memory pool
            times.append(max(e0.elapsed_time(e1) / 1000.0, 0.0) or wall)
        units = w.input_tuples() + (res.count if w.output_mode == "count" else 0)
    t = statistics.median(times)
    return {"value": units / t, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": 1000 * t, "steps": steps}


def e2e_leg_sharded(sharded, w, mv, steps, flush, world, backend):
    """N-rank end to end through the C-ABI: every rank's pinned host slice of
    each base relation -> fjg_relation_create (H2D) -> fjg_sharded_create ->
    fjg_execute_multi (partition + NCCL exchange + query + all-reduce, result
    on the host) -> destroy. Device-timed with CUDA events on the engine
    stream every call runs on, max over ranks."""
    import numpy as np
    import torch
    from paper_2301_10841_b200 import dist as D
    eng = sharded.engine
    stream = torch.cuda.ExternalStream(eng.stream_ptr, device=torch.device("cuda", eng.device))
    host = {b: [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in cols]
            for b, cols in sharded.local.items()}
    h2d = sum(t.numel() * 4 for cols in host.values() for t in cols)
    d2h = 8 * 7  # the reduced (count limbs, checksum halves, min) words
    times = []
    for i in range(steps + 1):
        eng.sync()
        barrier(world)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sq = D.ShardedQuery(eng, w, sharded.plan, sharded.comm, local=host)
        res = sq.execute(min_var=mv, output_mode=w.output_mode, backend=backend)
        e1.record(stream)
        eng.sync()
        sq.close()
        with torch.cuda.stream(stream):
            flush.add_(1)
        if i > 0:  # first iteration warms the memory pool
            times.append(e0.elapsed_time(e1) / 1000.0)
    t = allreduce_max(statistics.median(times), world)
    out_local = res.extra.get("local_count", res.count)
    units = allreduce_sum(sharded.input_tuples_local + (out_local if w.output_mode == "count" else 0), world)
    return {"value": units / t, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": 1000 * t, "steps": steps}


def main():
    args = parse()
    maybe_relaunch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
