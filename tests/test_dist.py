"""Multi-GPU exchange logic (paper_2301_10841_b200/dist.py) on CPU: world_size
2 and 3 over gloo. Each rank starts with a contiguous slice of every base
relation, runs the first-variable partition all-to-all + all-gather, executes
its shard with the oracle, and the all-reduced result must equal the
single-process oracle (count, checksum, MIN)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2301_10841_b200 import configs, dist as D, plan as P


def np_partition_of(v, nparts):
    """Vectorised fj::partition_of (fmix64(v ^ 0x5bd1e995) mod nparts)."""
    with np.errstate(over="ignore"):
        k = v.astype(np.int64).astype(np.uint64) ^ np.uint64(0x5bd1e995)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xff51afd7ed558ccd)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xc4ceb9fe1a85ec53)
        k ^= k >> np.uint64(33)
    return (k % np.uint64(nparts)).astype(np.int64)


class CpuOps:
    device = torch.device("cpu")

    def empty(self, n):
        return torch.empty(n, dtype=torch.int32)

    def partition(self, cols, col, world):
        dest = np_partition_of(cols[col].numpy(), world)
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest, minlength=world).tolist()
        return [torch.from_numpy(c.numpy()[order].copy()) for c in cols], counts


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = {"triangle": lambda: configs.triangle(scale=11, m=8000, seed=5),
             "chain": lambda: configs.chain(n=3000, domain=3000),
             "star": lambda: configs.star(nf=60000, dims=(2000, 3000, 800, 100)),
             "clique4": lambda: configs.clique4(scale=10, m=6000)}[name]()
        plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
        fv, views = D.atom_views(w.query, w.atom_rel, plan)
        local = {}
        for base, cols in w.filtered().items():
            lo, hi = D.local_slice(len(cols[0]), world, rank)
            local[base] = [torch.from_numpy(c[lo:hi].copy()) for c in cols]
        held = D.exchange(local, views, world, rank, CpuOps())
        cols = [[c.numpy() for c in held[v]] for v in views]
        head = P.head_variables(w.query)
        mv = head.index(w.min_var) if w.min_var else -1
        r = oracle.execute(w.query, plan, cols, min_var=mv)
        # every partitioned view must hold exactly this rank's first-variable values
        for (base, col), v in zip(views, views):
            if col is not None:
                assert (np_partition_of(held[v][col].numpy(), world) == rank).all()
        total, cs, mn = D.reduce_results(r["count"], r["checksum"], r["min"], torch.device("cpu"))
        if rank == 0:
            q.put((total, cs, mn))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["triangle", "chain", "star", "clique4"])
def test_sharded_equals_single(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    total, cs, mn = q.get(timeout=10)
    w = {"triangle": lambda: configs.triangle(scale=11, m=8000, seed=5),
         "chain": lambda: configs.chain(n=3000, domain=3000),
         "star": lambda: configs.star(nf=60000, dims=(2000, 3000, 800, 100)),
         "clique4": lambda: configs.clique4(scale=10, m=6000)}[name]()
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    head = P.head_variables(w.query)
    ref = oracle.execute(w.query, plan, w.atom_columns(), min_var=head.index(w.min_var) if w.min_var else -1)
    assert total == ref["count"] and cs == ref["checksum"] and mn == ref["min"]
    assert total > 0 or name == "star"


def test_np_partition_matches_oracle():
    v = np.array([0, 1, -1, 2**31 - 1, -2**31, 12345, 999999], dtype=np.int32)
    for n in (2, 3, 8):
        assert np_partition_of(v, n).tolist() == [oracle.partition_of(int(x), n) for x in v]


def test_reduce_results_carries():
    # 128-bit count and u64 checksum recombination without a process group
    big = (1 << 70) + 12345
    parts = [big & D.MASK32, (big >> 32) & D.MASK32, (big >> 64) & D.MASK32, big >> 96]
    assert parts[0] + (parts[1] << 32) + (parts[2] << 64) + (parts[3] << 96) == big


_NCCL_SCRIPT = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs, dist as D, plan as P
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
out = {}
for name, w in (("triangle", configs.triangle(scale=11, m=8000, seed=5)),
                ("star", configs.star(nf=60000, dims=(2000, 3000, 800, 100)))):
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    eng = fjg.Engine(0)
    sq = D.ShardedQuery(eng, w, plan, 1, 0)
    rs = [sq.execute(min_var=w.min_var, output_mode=w.output_mode) for _ in range(2)]
    out[name] = [[r.count, r.checksum, r.min_value] for r in rs]
dist.destroy_process_group()
print(json.dumps(out))
'''


@pytest.mark.gpu
def test_sharded_nccl_one_rank_matches_oracle(tmp_path):
    """The product exchange (CUDA partition kernel + NCCL all-to-all /
    all-gather, one all-gather of the size metadata, all-gathered result
    reduction) at world 1, run twice (persistent buffers reused), vs the oracle."""
    import subprocess
    import sys
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    got = __import__("json").loads(p.stdout.strip().splitlines()[-1])
    for name, w in (("triangle", configs.triangle(scale=11, m=8000, seed=5)),
                    ("star", configs.star(nf=60000, dims=(2000, 3000, 800, 100)))):
        plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
        head = P.head_variables(w.query)
        ref = oracle.execute(w.query, plan, w.atom_columns(), min_var=head.index(w.min_var) if w.min_var else -1)
        for c, cs, mn in got[name]:
            assert (c, cs, mn) == (ref["count"], ref["checksum"], ref["min"]), name
