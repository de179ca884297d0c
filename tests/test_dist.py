"""Multi-GPU exchange protocol on CPU: world_size 2 and 3 over gloo with the
protocol model (tests/dist_model.py, the steps of fjg_execute_multi). Each rank
starts with a contiguous slice of every base relation, runs the first-variable
partition all-to-all + all-gather, executes its shard with the oracle, and the
reduced result must equal the single-process oracle (count, checksum, MIN).
The product's C++ receive layout (fjg_exchange_layout) is checked against the
model; the product path itself (NCCL) runs at world 1 on the GPU, through
ctypes and from a compiled C++ caller."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import dist_model as D
from oracle import oracle
from paper_2301_10841_b200 import configs, plan as P
from paper_2301_10841_b200 import dist as PD


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
        fv, views = PD.atom_views(w.query, w.atom_rel, plan)
        local = {}
        for base, cols in w.filtered().items():
            lo, hi = PD.local_slice(len(cols[0]), world, rank)
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


def _gloo_one_rank(fn):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        return fn()
    finally:
        dist.destroy_process_group()


def test_reduce_results_carries():
    """The model's reduction at one rank: a count above 2^64 survives the 32-bit
    limb split, the checksum wraps mod 2^64, a missing MIN stays None."""
    big = (1 << 70) + 12345
    total, cs, mn = _gloo_one_rank(lambda: D.reduce_results(big, (1 << 64) - 3, None, torch.device("cpu")))
    assert total == big and cs == (1 << 64) - 3 and mn is None
    total, cs, mn = _gloo_one_rank(lambda: D.reduce_results(7, 5, -9, torch.device("cpu")))
    assert (total, cs, mn) == (7, 5, -9)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_exchange_layout_matches_model(world):
    """The C++ receive layout of fjg_execute_multi (fjg_exchange_layout) equals
    the protocol model's for random metadata, every rank, mixed view kinds."""
    import ctypes as C
    from paper_2301_10841_b200 import _capi
    rng = np.random.default_rng(world)
    nviews = 3
    part = [1, 0, 1]
    M = rng.integers(0, 1000, size=(world, nviews, world)).astype(np.uint64)
    for src in range(world):
        M[src, 1, :] = M[src, 1, 0]  # a replicated view repeats its row count
    for rank in range(world):
        off = np.zeros(nviews * world, dtype=np.uint64)
        rows = np.zeros(nviews, dtype=np.uint64)
        pv = (C.c_int * nviews)(*part)
        _capi.check(_capi.lib.fjg_exchange_layout(M.ctypes.data, nviews, world, rank, pv, off.ctypes.data,
                                                  rows.ctypes.data))
        moff, mrows = D.recv_layout(M.tolist(), part, rank)
        assert off.reshape(nviews, world).tolist() == moff and rows.tolist() == mrows


_NCCL_SCRIPT = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs, dist as D, plan as P
out = {}
eng = fjg.Engine(0)
comm = D.Comm(eng, 1, 0)
for name, w in (("triangle", configs.triangle(scale=11, m=8000, seed=5)),
                ("star", configs.star(nf=60000, dims=(2000, 3000, 800, 100))),
                ("path5", configs.path5(scale=10, m=6000))):
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    sq = D.ShardedQuery(eng, w, plan, comm)
    rs = [sq.execute(min_var=w.min_var, output_mode=w.output_mode, timing=True) for _ in range(2)]
    out[name] = [[r.count, r.checksum, r.min_value, r.extra["local_count"]] for r in rs]
    sq.close()
comm.close()
print(json.dumps(out))
'''


@pytest.mark.gpu
def test_sharded_nccl_one_rank_matches_oracle(tmp_path):
    """The product multi-GPU path (fjg_execute_multi: CUDA partition kernel,
    NCCL metadata all-gather, grouped send/recv, all-reduce) at world 1, run
    twice (persistent buffers reused), vs the oracle."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", _NCCL_SCRIPT], cwd=root, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    got = __import__("json").loads(p.stdout.strip().splitlines()[-1])
    for name, w in (("triangle", configs.triangle(scale=11, m=8000, seed=5)),
                    ("star", configs.star(nf=60000, dims=(2000, 3000, 800, 100))),
                    ("path5", configs.path5(scale=10, m=6000))):
        plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
        head = P.head_variables(w.query)
        ref = oracle.execute(w.query, plan, w.atom_columns(), min_var=head.index(w.min_var) if w.min_var else -1,
                             output_mode=w.output_mode)
        for c, cs, mn, lc in got[name]:
            assert (c, mn) == (ref["count"], ref["min"]) and lc == c, name
            if w.output_mode == "count":
                assert cs == ref["checksum"], name
