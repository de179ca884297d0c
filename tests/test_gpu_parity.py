"""GPU parity: the sm_100a executor behind the C-ABI against the CPU oracle
(bit-exact count, checksum, MIN; bag equality in enumerate mode)."""
import json
import os

import numpy as np
import pytest

import paper_2301_10841_b200 as fjg
from oracle import oracle
from paper_2301_10841_b200 import configs, plan as P

from randq import bag_equal, random_query

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "configs_full.json")


def gpu_execute(engine, q, plan, cols, shared=None, **kw):
    """Bind one device relation per atom (or per shared group) and execute."""
    rels, keep = [], {}
    for i, c in enumerate(cols):
        key = shared[i] if shared else i
        if key not in keep:
            keep[key] = engine.relation(c)
        rels.append(keep[key])
    qq = engine.query({"query": q["query"] if isinstance(q, dict) else q}, plan, rels)
    if kw.pop("enumerate", False):
        rows, r = qq.enumerate(**kw)
        return r, rows
    return qq.execute(**kw), None


def check(engine, q, plan, cols, shared=None, enumerate=False, min_var=None, **kw):
    ref = oracle.execute(q, plan, cols, output_mode="enumerate" if enumerate else "count",
                         min_var=-1 if min_var is None else min_var, dynamic_cover=kw.get("dynamic_cover", True))
    r, rows = gpu_execute(engine, q, plan, cols, shared=shared, enumerate=enumerate, min_var=min_var, **kw)
    assert r.count == ref["count"], (r.count, ref["count"])
    assert r.checksum == ref["checksum"], (hex(r.checksum), hex(ref["checksum"]))
    if min_var is not None:
        assert r.min_value == ref["min"]
    if enumerate:
        assert bag_equal(rows, ref["tuples"])
    return r, ref


@pytest.mark.parametrize("block", range(3))
def test_random_queries(engine, block):
    """SPEC.md:434 property: random skewed instances with duplicates, all plan modes."""
    rng = np.random.default_rng(4242 + block)
    n = 0
    while n < 40:
        q, cols = random_query(rng)
        if len(oracle.brute_force(q, cols)) > 50000:
            continue
        n += 1
        for mode in ("binary", "free", "generic"):
            plan = P.compile_plan(q, mode)
            dyn = bool(rng.random() < 0.7)
            batch = int(rng.choice([0, 3, 7, 1000]))
            backend = str(rng.choice(["colt", "colt", "slt", "simple"]))
            check(engine, q, plan, cols, enumerate=(n % 4 == 0), dynamic_cover=dyn, batch_size=batch,
                  backend=backend)


def test_self_joins_share_tries(engine):
    """Renamed self-joins bound to one relation share physical COLT levels."""
    rng = np.random.default_rng(77)
    for _ in range(25):
        nv = int(rng.integers(3, 6))
        pool = [f"v{i}" for i in range(nv)]
        natoms = int(rng.integers(2, 5))
        q = {"query": [{"rel": f"E{a}", "vars": [str(x) for x in rng.choice(pool, 2, replace=False)]}
                       for a in range(natoms)]}
        dom = int(rng.integers(3, 12))
        E = [rng.integers(0, dom, 40).astype(np.int32), rng.integers(0, dom, 40).astype(np.int32)]
        cols = [E] * natoms
        for mode in ("free", "generic"):
            check(engine, q, P.compile_plan(q, mode), cols, shared=[0] * natoms)


def test_edge_cases(engine):
    tri = [{"rel": "R", "vars": ["x", "y"]}, {"rel": "S", "vars": ["y", "z"]}, {"rel": "T", "vars": ["x", "z"]}]
    e = np.zeros(0, np.int32)
    one = [np.array([1], np.int32), np.array([2], np.int32)]
    dup = [np.array([1, 1, 1, 2], np.int32), np.array([2, 2, 2, 3], np.int32)]
    ext = [np.array([-2**31, 2**31 - 1, 0, -1], np.int32), np.array([2**31 - 1, -2**31, -1, 0], np.int32)]
    for mode in ("binary", "free", "generic"):
        plan = P.compile_plan(tri, mode)
        check(engine, tri, plan, [[e, e], one, one])                 # empty relation
        check(engine, tri, plan, [one, [one[1], one[1]], one])       # single rows
        check(engine, tri, plan, [dup, [dup[1], dup[1]], dup], enumerate=True)  # multiplicities
        check(engine, tri, plan, [ext, ext, ext], enumerate=True)    # int32 extremes
    # Cartesian product (empty-vars probe subatoms) and arity-2 probe keys
    cart = [{"rel": "A", "vars": ["x"]}, {"rel": "B", "vars": ["y"]}, {"rel": "C", "vars": ["x", "y"]}]
    cc = [[np.array([1, 2, 2], np.int32)], [np.array([5, 6], np.int32)],
          [np.array([1, 2, 2, 3], np.int32), np.array([5, 6, 6, 5], np.int32)]]
    for mode in ("binary", "free", "generic"):
        check(engine, cart, P.compile_plan(cart, mode), cc, enumerate=True)
    wide = [{"rel": "R", "vars": ["a", "b", "c"]}, {"rel": "S", "vars": ["a", "b", "c", "d"]}]
    rng = np.random.default_rng(3)
    wc = [[rng.integers(0, 3, 60).astype(np.int32) for _ in range(3)],
          [rng.integers(0, 3, 60).astype(np.int32) for _ in range(4)]]
    check(engine, wide, P.compile_plan(wide, "binary"), wc, enumerate=True)  # arity-3 probe key


def test_batch_and_cover_invariance(engine):
    w = configs.triangle(scale=11, m=12000, seed=9)
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    ref = oracle.execute(w.query, plan, w.atom_columns())
    for batch in (0, 1000, 7777):
        for dyn in (True, False):
            r, _ = gpu_execute(engine, {"query": w.query}, plan, w.atom_columns(), shared=[0, 0, 0],
                               batch_size=batch, dynamic_cover=dyn)
            assert (r.count, r.checksum) == (ref["count"], ref["checksum"])


@pytest.mark.parametrize("name", ["chain", "triangle", "star", "clique4"])
def test_configs_small(engine, name):
    small = {"chain": lambda: configs.chain(n=50000, domain=50000),
             "triangle": lambda: configs.triangle(scale=14, m=200000, seed=3),
             "star": lambda: configs.star(nf=2_000_000, dims=(40000, 60000, 16000, 2000)),
             "clique4": lambda: configs.clique4(scale=14, m=150000)}[name]()
    res, q, plan, _ = fjg.run_workload(engine, small)
    mv = q.head.index(small.min_var) if small.min_var else -1
    ref = oracle.execute(small.query, plan, small.atom_columns(), min_var=mv, nthreads=os.cpu_count() or 1)
    assert (res.count, res.checksum) == (ref["count"], ref["checksum"])
    if small.min_var:
        assert res.min_value == ref["min"]
    assert res.kernel_launches > 0


def _golden(name):
    if not os.path.exists(GOLDEN):
        pytest.skip("no golden file")
    g = json.load(open(GOLDEN))
    if name not in g:
        pytest.skip(f"no golden for {name}")
    return g[name]


@pytest.mark.parametrize("name", ["chain", "triangle", "star", "clique4"])
def test_configs_full_vs_golden(engine, name):
    """BASELINE.json configs at full size vs the oracle's committed results."""
    g = _golden(name)
    w = configs.CONFIGS[name]()
    assert w.params == g["params"]
    res, q, plan, _ = fjg.run_workload(engine, w)
    assert [[(r, list(v)) for (r, v) in n] for n in plan] == [[(r, list(v)) for (r, v) in n] for n in g["plan"]]
    assert res.count == g["count"]
    assert f"{res.checksum:#018x}" == g["checksum"]
    if w.min_var:
        assert res.min_value == g["min"]


def test_chain_full_sorted_output(engine):
    """C1: full materialised output compared with the oracle's (sorted)."""
    w = configs.chain()
    q, plan, _ = fjg.prepare_workload(engine, w)
    rows, r = q.enumerate()
    ref = oracle.execute(w.query, plan, w.atom_columns(), output_mode="enumerate", nthreads=os.cpu_count() or 1)
    assert r.count == len(rows) == ref["count"]
    assert bag_equal(rows, ref["tuples"])


def test_filter_and_partition_kernels(engine):
    rng = np.random.default_rng(1)
    c0 = rng.integers(-1000, 1000, 100000).astype(np.int32)
    c1 = rng.integers(-1000, 1000, 100000).astype(np.int32)
    rel = engine.relation([c0, c1])
    f = rel.filter([(0, "<", 10), (1, ">=", -500)]).download()
    keep = (c0 < 10) & (c1 >= -500)
    assert (f[0] == c0[keep]).all() and (f[1] == c1[keep]).all()
    g = rel.filter([(0, "=", ("col", 1))]).download()
    assert (g[0] == c0[c0 == c1]).all()
    for G in (4, 3, 8, 1):  # the power-of-two mask path and the modulo path
        part, counts = rel.partition(0, G)
        cols = part.download()
        dest = np.array([oracle.partition_of(v, G) for v in c0])
        off = 0
        for d in range(G):
            assert counts[d] == int((dest == d).sum())
            assert (cols[0][off:off + counts[d]] == c0[dest == d]).all()  # stable within a destination
            assert (cols[1][off:off + counts[d]] == c1[dest == d]).all()
            off += counts[d]


def test_int64_columns_narrowed_on_device(engine):
    """fjg_relation_create_i64 (fj::Value is int64, value.hpp:31): int64 host columns give the same relation,
    and the same query result, as their int32 copies; a value outside int32 is a ValidationError naming it."""
    rng = np.random.default_rng(7)
    for n in (0, 1, 3, 4, 5, 1000, 100003):
        c0 = rng.integers(-2**31, 2**31, n, dtype=np.int64)
        c1 = rng.integers(-5, 5, n, dtype=np.int64)
        got = engine.relation_i64([c0, c1]).download()
        assert (got[0] == c0.astype(np.int32)).all() and (got[1] == c1.astype(np.int32)).all()
    w = configs.triangle(scale=10, m=8000, seed=2)
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    cols = w.atom_columns()
    ref = oracle.execute(w.query, plan, cols)
    rel = engine.relation_i64([np.asarray(c, dtype=np.int64) for c in cols[0]])
    r = engine.query({"query": w.query}, plan, [rel] * 3).execute()
    assert (r.count, r.checksum) == (ref["count"], ref["checksum"])
    bad = np.arange(10, dtype=np.int64)
    for v, row in ((2**31, 6), (-2**31 - 1, 9), (2**40, 0)):
        b = bad.copy()
        b[row] = v
        with pytest.raises(fjg.ValidationError, match=f"column 1, row {row}"):
            engine.relation_i64([bad, b])


def test_optimistic_force_redo_on_repeated_keys(engine):
    """Level >= 1 forces insert optimistically (every key of a subtrie distinct) and redo a member with the
    counting protocol when a repeated key shows up: a multigraph triangle whose early subtries are duplicate
    free and whose later ones repeat keys, under small batches (several force batches per execution: optimistic,
    then redo, then the level's dup flag routes later batches to the counting protocol), executed twice."""
    rng = np.random.default_rng(11)
    n = 6000
    src = rng.integers(0, 300, n).astype(np.int32)
    dst = rng.integers(0, 300, n).astype(np.int32)
    clean = np.unique(np.stack([src, dst], 1), axis=0)  # duplicate-free prefix ...
    dup = clean[rng.integers(len(clean) // 2, len(clean), 2000)]  # ... then repeats of the upper half
    e = np.concatenate([clean, dup])
    cols = [np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])]
    q = [{"rel": "E1", "vars": ["a", "b"]}, {"rel": "E2", "vars": ["b", "c"]}, {"rel": "E3", "vars": ["a", "c"]}]
    plan = P.compile_plan({"query": q, "binary_plan": configs.left_deep(["E1", "E2", "E3"])}, "generic")
    for dyn in (True, False):
        for bs in (0, 997, 64):
            r, ref = check(engine, q, plan, [cols] * 3, shared=[0, 0, 0], dynamic_cover=dyn, batch_size=bs)
            assert r.count > 0
    rel = engine.relation(cols)
    qq = engine.query({"query": q}, plan, [rel] * 3)
    a, b = qq.execute(batch_size=500), qq.execute(batch_size=500)
    assert (a.count, a.checksum) == (b.count, b.checksum)


def test_counters(engine):
    """ExecStats: probes/misses/body entries agree with the oracle where forcing order is pinned (chain)."""
    w = configs.chain(n=20000, domain=30000)
    res, q, plan, _ = fjg.run_workload(engine, w)
    ref = oracle.execute(w.query, plan, w.atom_columns())
    assert res.probes == ref["probes"]
    assert res.probe_misses == ref["probe_misses"]
    assert res.node_body_entries == ref["node_body_entries"][:len(plan)]
    assert res.maps_built >= 2  # S and T roots forced, R never (BaseScan)


def test_device_rmat_matches_host():
    from paper_2301_10841_b200 import datagen
    import torch
    s, d = datagen.rmat(21, 14, 200000)
    ds, dd = datagen.rmat_device(21, 14, 200000)
    assert (ds.cpu().numpy() == s).all() and (dd.cpu().numpy() == d).all()
    torch.cuda.synchronize()


@pytest.fixture
def own_engine():
    """A private engine for the full-size tests: closing it returns its memory
    pool (tens of GB at 2^27) before the next test allocates."""
    import torch
    eng = fjg.Engine(0)
    yield eng
    eng.close()
    torch.cuda.empty_cache()


def test_scale_triangle_partition(own_engine):
    """C5 at full size (R-MAT 2^27, 512M edges): the first-variable hash
    partition r of G (E1, E3 restricted, E2 whole) vs the oracle's committed
    result (tests/golden/make_scale_goldens.py)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "scale_partition.json")
    if not os.path.exists(path):
        pytest.skip("no scale golden")
    g = json.load(open(path))
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_scale_goldens import restricted
    w = configs.scale_triangle()
    assert w.params == g["params"]
    cols = restricted(w)
    assert len(cols[0][0]) == g["rows_partition"]
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    engine = own_engine
    part = engine.relation(cols[0])
    full = engine.relation(cols[1])
    r = engine.query({"query": w.query}, plan, [part, full, part]).execute()
    assert r.count == g["count"] and f"{r.checksum:#018x}" == g["checksum"]


@pytest.mark.parametrize("scale,m", [(8, 1500), (12, 30000), (16, 400000)])
def test_path5_memoised_count(engine, scale, m):
    """C5 5-path at reduced scale: the device memoised chain count equals the
    oracle's memoised count and an independent exact 1^T A^5 1."""
    w = configs.path5(scale=scale, m=m, seed=5)
    res, q, plan, _ = fjg.run_workload(engine, w, output_mode="factorized_count")
    ref = oracle.execute(w.query, plan, w.atom_columns(), output_mode="factorized_count")
    assert ref["factorized"]
    src, dst = w.relations["E"]
    x = np.ones(1 << scale, dtype=object)
    for _ in range(5):
        y = np.zeros(1 << scale, dtype=object)
        np.add.at(y, src, x[dst])
        x = y
    assert res.count == ref["count"] == int(x.sum())
    if scale == 8:  # plain enumeration agrees too
        assert fjg.run_workload(engine, w)[0].count == res.count


def test_scale_triangle_full_vs_golden(own_engine):
    """C5 triangle at full size (R-MAT 2^27, 512M edges, ~4.1e9 triangles):
    count and checksum vs tests/golden/configs_full.json["scale_triangle"]
    (tests/golden/make_xcheck_goldens.py: the independent CSR counter, which
    agrees with the oracle on C2, C4 and on C5 partition 0 of 256)."""
    g = _golden("scale_triangle")
    w = configs.scale_triangle()
    assert w.params == g["params"]
    res, q, plan, rels = fjg.run_workload(own_engine, w)
    assert [[[r, list(v)] for (r, v) in n] for n in plan] == g["plan"]
    assert res.count == g["count"]
    assert f"{res.checksum:#018x}" == g["checksum"]


def test_scale_path5_exact_vs_golden(own_engine):
    """C5 5-path at full size: the device memoised count equals the exact walk
    count 1^T A^5 1 (xcheck SpMV residues mod 2^64 and two 61-bit primes,
    combined by CRT) committed in configs_full.json["scale_path5"]."""
    g = _golden("scale_path5")
    w = configs.scale_path5()
    assert w.params == g["params"]
    res, q, plan, rels = fjg.run_workload(own_engine, w)
    assert res.count == g["count"]


def test_scale_path5_residues(own_engine):
    """C5 5-path at full size (~4.9e21 walks, > 2^64): the device memoised count
    agrees with 1^T A^5 1 computed independently by torch index_add SpMV,
    modulo 2^64 and modulo two primes (exact integer residues)."""
    import torch
    w = configs.scale_path5()
    res, q, plan, rels = fjg.run_workload(own_engine, w)
    assert res.count > 2 ** 64
    q.close()
    for r in rels.values():
        r.close()
    own_engine.close()  # return the pool before the torch SpMV below
    torch.cuda.empty_cache()
    src = torch.from_numpy(w.relations["E"][0]).cuda().long()
    dst = torch.from_numpy(w.relations["E"][1]).cuda().long()
    n = 1 << w.params["scale"]
    for mod in (None, 2_147_483_647, 1_000_000_007):
        x = torch.ones(n, dtype=torch.int64, device="cuda")
        for _ in range(5):
            y = torch.zeros(n, dtype=torch.int64, device="cuda")
            y.index_add_(0, src, x[dst])  # wraps mod 2^64 when mod is None
            x = y if mod is None else y % mod
        tot = int(x.sum().item()) if mod is not None else int(x.sum().item()) & (2 ** 64 - 1)
        if mod is None:
            assert tot == res.count % 2 ** 64
        else:
            assert tot % mod == res.count % mod


def test_run_segments_bushy(engine):
    """SPEC acceptance #7: bushy trees decompose into segments whose
    device-materialised results feed the parent; output == brute force."""
    from paper_2301_10841_b200.segments import run_segments
    rng = np.random.default_rng(31)
    trees = [["join", ["join", "A0", "A1"], ["join", "A2", "A3"]],
             ["join", "A0", ["join", "A1", ["join", "A2", "A3"]]],
             ["join", ["join", "A0", ["join", "A1", "A2"]], "A3"]]
    done = 0
    while done < 24:
        q, cols = random_query(rng, max_atoms=4)
        if len(q["query"]) != 4:
            continue
        truth = oracle.brute_force(q, cols)
        if len(truth) > 20000:
            continue
        done += 1
        rels = {a["rel"]: engine.relation(c) for a, c in zip(q["query"], cols)}
        for tree in trees:
            for mode in ("free", "generic"):
                try:
                    r, qq, trace = run_segments(engine, q["query"], tree, rels, mode=mode, output_mode="enumerate")
                except fjg.ResourceError:
                    continue  # a segment wider than 8 variables
                assert bag_equal(r.extra["rows"], truth), (tree, mode)
                assert r.checksum == oracle.checksum_of(truth)
                assert len(trace) == len(P.decompose_bushy(tree, q["query"]))


def test_empty_root_after_reuse(engine):
    """A 0-row relation probed after its trie memory held an earlier query's
    slots must miss (regression: stale buckets of an empty region)."""
    q = [{"rel": "A", "vars": ["x", "y"]}, {"rel": "B", "vars": ["x"]}]
    plan = P.compile_plan(q, "free")
    a = [np.arange(100, dtype=np.int32) % 7, np.arange(100, dtype=np.int32)]
    for _ in range(3):
        big = engine.query({"query": q}, plan, [engine.relation(a), engine.relation([a[0]])])
        assert big.execute().count > 0
        big.close()
        empty = engine.query({"query": q}, plan, [engine.relation(a), engine.relation([np.zeros(0, np.int32)])])
        assert empty.execute().count == 0
        empty.close()


def test_backend_ladder(engine):
    """GHT backends on the device (acceptance #5, the §5.3
    ladder): identical outputs; keys_inserted colt <= slt <= simple with
    colt < simple; the eager SIMPLE build inserts exactly the oracle's keys."""
    rng = np.random.default_rng(5)
    n = 100_000
    zipf = lambda: np.minimum(rng.zipf(1.3, n) - 1, 5000).astype(np.int32)  # noqa: E731
    uni = lambda: rng.integers(0, 100_000_000, n).astype(np.int32)  # noqa: E731
    q = [{"rel": "R", "vars": ["x", "y"]}, {"rel": "S", "vars": ["y", "z"]}, {"rel": "T", "vars": ["x", "z"]}]
    cols = [[zipf(), uni()], [uni(), zipf()], [zipf(), zipf()]]
    plan = P.compile_plan(q, "generic")
    rels = [engine.relation(c) for c in cols]
    query = engine.query({"query": q}, plan, rels)
    dev = {b: query.execute(backend=b) for b in ("colt", "slt", "simple")}
    ref = {b: oracle.execute(q, plan, cols, backend=b) for b in ("colt", "simple")}
    for b, r in dev.items():
        assert r.count == ref["colt"]["count"] and r.checksum == ref["colt"]["checksum"], b
    k = {b: r.keys_inserted for b, r in dev.items()}
    assert k["colt"] <= k["slt"] <= k["simple"] and k["colt"] < k["simple"]
    assert k["simple"] == ref["simple"]["keys_inserted"]
    # enumerate through an eager backend: same bag as the lazy one
    t_colt, _ = query.enumerate(backend="colt")
    t_simple, _ = query.enumerate(backend="simple")
    assert sorted(map(tuple, t_colt.tolist())) == sorted(map(tuple, t_simple.tolist()))


@pytest.mark.parametrize("name", ["chain", "triangle", "clique4"])
def test_backends_configs(engine, name):
    """Eager backends on reduced configs (shared physical tries, leaf levels):
    same count and checksum as COLT and the oracle."""
    w = {"chain": lambda: configs.chain(n=20000, domain=20000),
         "triangle": lambda: configs.triangle(scale=12, m=30000, seed=3),
         "clique4": lambda: configs.clique4(scale=12, m=40000)}[name]()
    q, plan, _ = fjg.prepare_workload(engine, w)
    ref = oracle.execute(w.query, plan, w.atom_columns())
    for b in ("colt", "slt", "simple"):  # noqa: B007
        r = q.execute(backend=b)
        assert (r.count, r.checksum) == (ref["count"], ref["checksum"]), b


def _fmix32(h):
    h = np.asarray(h, dtype=np.uint64) & 0xFFFFFFFF
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & 0xFFFFFFFF
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & 0xFFFFFFFF
    h ^= h >> 16
    return h


def _colliding_keys(rng, length, bucket, n, exclude=()):
    """n int32 keys whose first bucket inside a `length`-bucket region is
    `bucket` (region_bucket in kernels/common.cuh)."""
    out = []
    while len(out) < n:
        k = rng.integers(-2**31, 2**31, 4096, dtype=np.int64)
        off = (_fmix32((k & 0xFFFFFFFF) ^ 0x9E3779B9) * length) >> 32
        out.extend(int(x) for x in k[off == bucket] if int(x) not in exclude and int(x) not in out)
    return out[:n]


def test_bucket_collisions_and_extreme_keys(engine):
    """Adversarial probes for the last-node kernels: 40 keys of one subtrie
    all hashed to its last bucket (a 10-bucket overflow chain that wraps to
    the region start), misses that walk the whole chain, and the int32
    extremes (INT32_MIN, INT32_MAX, -1 whose key word equals the empty
    marker, 0) as vertices -- every plan mode and backend vs the oracle."""
    rng = np.random.default_rng(99)
    A, B, C = 7, 11, 13
    extremes = [-2**31, 2**31 - 1, -1, 0]
    sa = _colliding_keys(rng, 48, 47, 44, exclude=[A, B, C] + extremes)     # A's region: 48 rows
    sa = sa[:44] + [B, C] + extremes[:2]                                   # 48 out-neighbours of A
    miss = _colliding_keys(rng, 48, 47, 6, exclude=sa + [A] + extremes)    # collide with A's chain, absent
    tb = sa[:3] + sa[-6:-2] + miss + extremes                              # B: hits, misses, extremes
    tc = sa[10:30] + miss[:2]                                              # C: longer list
    edges = [(A, x) for x in sa] + [(B, x) for x in tb] + [(C, x) for x in tc]
    edges += [(x, y) for x, y in zip(extremes, reversed(extremes)) if x != y]
    edges += [(int(x), int(y)) for x, y in rng.integers(-50, 50, (300, 2)) if x != y]
    edges = sorted(set(edges))
    order = rng.permutation(len(edges))
    src = np.array([edges[i][0] for i in order], np.int32)
    dst = np.array([edges[i][1] for i in order], np.int32)
    q = [{"rel": "E1", "vars": ["a", "b"]}, {"rel": "E2", "vars": ["b", "c"]}, {"rel": "E3", "vars": ["a", "c"]}]
    cols = [[src, dst]] * 3
    rel = engine.relation([src, dst])
    for mode in ("binary", "free", "generic"):
        plan = P.compile_plan({"query": q, "binary_plan": ["join", ["join", "E1", "E2"], "E3"]}, mode)
        ref = oracle.execute(q, plan, cols, output_mode="enumerate")
        qq = engine.query({"query": q}, plan, [rel, rel, rel])
        for backend in ("colt", "simple"):
            r = qq.execute(backend=backend)
            assert (r.count, r.checksum) == (ref["count"], ref["checksum"]), (mode, backend)
        rows, _ = qq.enumerate()
        assert bag_equal(rows, ref["tuples"])
        qq.close()
    assert ref["count"] > 0


@pytest.mark.parametrize("ndims", [1, 2, 3, 4])
def test_stream_one_and_cartesian_tail(engine, ndims):
    """Factored star plans: node 0 streams the fact table and probes every
    dimension (k_stream_one: stage queues, NP = ndims); the per-dimension
    suffix nodes form a Cartesian tail (k_tail) whose products exceed 8 rows
    per binding (warp-strided expansion). Count, checksum, MIN and the
    enumerated bag match the oracle for batch sizes that split node 0."""
    rng = np.random.default_rng(900 + ndims)
    nf = 3000
    q = [{"rel": "F", "vars": ["r"] + [f"f{i + 1}" for i in range(ndims)]}]
    cols = [[np.arange(nf, dtype=np.int32)] + [rng.integers(0, 40, nf).astype(np.int32) for _ in range(ndims)]]
    for i in range(ndims):
        keys = rng.integers(0, 60, 90).astype(np.int32)      # duplicate keys: tails of several rows
        if i == 0:
            keys = np.concatenate([keys, np.full(12, 7, np.int32)])  # one key with > 8 rows
        q.append({"rel": f"D{i + 1}", "vars": [f"f{i + 1}", f"x{i + 1}"]})
        cols.append([keys, rng.integers(-5, 5, len(keys)).astype(np.int32)])
    plan = P.compile_plan({"query": q, "binary_plan": configs.left_deep([a["rel"] for a in q])}, "free")
    assert len(plan) == ndims + 1 and all(len(node) == 1 for node in plan[1:])
    for batch in (0, 1000, 777):
        check(engine, q, plan, cols, min_var=0, batch_size=batch)
    check(engine, q, plan, cols, enumerate=True, batch_size=777)


def test_batched_root_forces_count_keys(engine):
    """Roots claimed together are forced in one batch (blockIdx.y = member):
    every backend's keys_inserted equals the oracle's (SLT / SIMPLE force all
    four dimension roots and the fact table's levels at once)."""
    rng = np.random.default_rng(31)
    q = [{"rel": "F", "vars": ["r", "f1", "f2", "f3"]}]
    cols = [[np.arange(500, dtype=np.int32)] + [rng.integers(0, 30, 500).astype(np.int32) for _ in range(3)]]
    for i in range(3):
        q.append({"rel": f"D{i + 1}", "vars": [f"f{i + 1}", f"x{i + 1}"]})
        keys = rng.integers(0, 40, 70).astype(np.int32)
        cols.append([keys, rng.integers(0, 9, 70).astype(np.int32)])
    plan = P.compile_plan({"query": q, "binary_plan": configs.left_deep([a["rel"] for a in q])}, "free")
    for backend in ("colt", "slt", "simple"):
        ref = oracle.execute(q, plan, cols, backend=backend)
        r, _ = gpu_execute(engine, q, plan, cols, backend=backend)
        assert (r.count, r.checksum) == (ref["count"], ref["checksum"])
        assert r.keys_inserted == ref["keys_inserted"], (backend, r.keys_inserted, ref["keys_inserted"])


def test_sorted_root_key_widths(engine):
    """Roots of >= 2^21 rows are forced by a radix sort over the key column's
    used bits (its maximum, computed at query creation): narrow, wide and
    negative keys (all 32 bits as uint32) give the oracle's results."""
    rng = np.random.default_rng(5)
    n = (1 << 21) + 77
    q = [{"rel": "E", "vars": ["a", "b"]}, {"rel": "S", "vars": ["b", "c"]}]
    for lo, hi in ((0, 1 << 20), (-(1 << 31), (1 << 31) - 1), (-(1 << 20), 1 << 20)):
        E = [rng.integers(0, 50, n).astype(np.int32), rng.integers(lo, hi, n, dtype=np.int64).astype(np.int32)]
        S = [np.concatenate([E[1][:3000], rng.integers(lo, hi, 100, dtype=np.int64).astype(np.int32)]),
             rng.integers(0, 7, 3100).astype(np.int32)]
        plan = P.compile_plan({"query": q, "binary_plan": configs.left_deep(["S", "E"])}, "free")
        check(engine, q, plan, [E, S])


def test_simple_backend_empty_relation_after_pool_reuse(engine):
    """SIMPLE forces every map level eagerly; an empty relation has no subtries
    below its root, and its deeper tables (recycled device memory) must not be
    read. The same query first runs with the relation non-empty so its freed
    tables hold occupied slots when the empty one is bound."""
    q = {"query": [{"rel": "A", "vars": ["x", "y", "z"]}, {"rel": "B", "vars": ["z", "x", "y"]},
                   {"rel": "C", "vars": ["y", "z"]}]}
    rng = np.random.default_rng(8)
    full = [rng.integers(0, 4, 24).astype(np.int32) for _ in range(3)]
    empty = [np.zeros(0, np.int32)] * 3
    C = [rng.integers(0, 4, 10).astype(np.int32) for _ in range(2)]
    for mode in ("generic", "free"):
        plan = P.compile_plan(q, mode)
        for b_cols in (full, empty, full, empty):
            cols = [[c.copy() for c in full], [c.copy() for c in b_cols], C]
            ref = oracle.execute(q, plan, cols, backend="simple", dynamic_cover=False)
            r, _ = gpu_execute(engine, q, plan, cols, backend="simple", dynamic_cover=False)
            assert (r.count, r.checksum, r.keys_inserted) == (ref["count"], ref["checksum"], ref["keys_inserted"])


def test_acceptance4_device_colt_laziness(engine):
    """SPEC acceptance #4 on the device: on the factored clover
    with COLT, R (the cover, BaseScan) builds no map and S / T force at most
    one level each; the extended clover with S(b) as cover builds no level-1
    map for S (Example 4.4)."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_acceptance import clover
    for n in (20, 2000):
        q, cols = clover(n)
        plan = P.compile_plan(q, "free")
        r, _ = gpu_execute(engine, q, plan, cols)
        ref = oracle.execute(q, plan, cols)
        assert r.count == ref["count"] == 1
        assert r.atom_maps_built[0] == 0 and r.atom_levels_forced[0] == 0  # R: BaseScan only
        for a in (1, 2):
            assert bin(r.atom_levels_forced[a]).count("1") <= 1
    q, cols = clover(20)
    q2 = q + [{"rel": "U", "vars": ["b"]}]
    U = [np.array([200, 3001, 3002], np.int32)]
    plan = [[("R", ["x", "a"]), ("S", ["x"]), ("T", ["x"])], [("S", ["b"]), ("U", ["b"])], [("T", ["c"])]]
    r, _ = gpu_execute(engine, q2, plan, cols + [U], dynamic_cover=False)
    assert r.count == 1
    assert not (r.atom_levels_forced[1] >> 1) & 1


def test_acceptance6_device_probe_counters_batch_invariant(engine):
    """SPEC acceptance #6 on the device: under a static cover the
    output bag and the probe counters do not depend on the batch size
    (1, 2, 7, 1000), and equal the oracle's."""
    rng = np.random.default_rng(66)
    done = 0
    while done < 12:
        q, cols = random_query(rng, max_atoms=4, max_rows=40)
        plan = P.compile_plan(q, "free")
        ref = oracle.execute(q, plan, cols, dynamic_cover=False, output_mode="enumerate")
        if ref["count"] > 5000:
            continue
        done += 1
        seen = None
        for b in (1, 2, 7, 1000):
            r, rows = gpu_execute(engine, q, plan, cols, batch_size=b, dynamic_cover=False, enumerate=True)
            assert bag_equal(rows, ref["tuples"])
            key = (r.probes, r.probe_misses, tuple(r.node_probes))
            seen = seen or key
            assert key == seen, (b, key, seen)
        assert seen[0] == ref["probes"]


_SORTED_SCRIPT = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs
eng = fjg.Engine(0)
out = []
for w in (configs.triangle(scale=12, m=40000, seed=4), configs.triangle(scale=14, m=200000, seed=8)):
    for batch in (0, 5000):
        res, q, plan, rels = fjg.run_workload(eng, w, batch_size=batch)
        out.append([res.count, res.checksum])
print(json.dumps(out))
'''


def test_gj_last_node_probe_region_order():
    """The GJ last node visiting bindings in probe-region order (the path C5
    takes, forced here on small inputs with FJG_GJ_SORT_MIN_ROWS=0) gives the
    oracle's count and checksum, for one and several frontier batches."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FJG_GJ_SORT_MIN_ROWS="0")
    p = subprocess.run([sys.executable, "-c", _SORTED_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    got = json.loads(p.stdout.strip().splitlines()[-1])
    i = 0
    for w in (configs.triangle(scale=12, m=40000, seed=4), configs.triangle(scale=14, m=200000, seed=8)):
        plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
        ref = oracle.execute(w.query, plan, w.atom_columns())
        for _ in range(2):
            assert got[i] == [ref["count"], ref["checksum"]]
            i += 1


def test_enumerate_single_pass_and_regrow(engine):
    """Enumerate is one pass that folds count / checksum too; an output larger
    than the buffer's capacity (2 x the largest relation at first) is rerun
    once at the exact size, and the capacity is kept for the next execution."""
    n = 700
    R = [np.arange(n, dtype=np.int32), np.zeros(n, np.int32)]
    S = [np.zeros(n, np.int32), np.arange(n, dtype=np.int32) + 5]
    q = [{"rel": "R", "vars": ["a", "b"]}, {"rel": "S", "vars": ["b", "c"]}]
    plan = P.compile_plan(q, "free")
    ref = oracle.execute(q, plan, [R, S], output_mode="enumerate")
    assert ref["count"] == n * n
    rels = [engine.relation(R), engine.relation(S)]
    qq = engine.query({"query": q}, plan, rels)
    for _ in range(2):  # first: regrow and rerun; second: the kept capacity fits
        rows, r = qq.enumerate()
        assert r.count == len(rows) == n * n and r.checksum == ref["checksum"]
        assert bag_equal(rows, ref["tuples"])
    c = qq.execute()
    assert (c.count, c.checksum) == (r.count, r.checksum)


@pytest.mark.parametrize("name", ["triangle", "clique4"])
def test_gj_last_node_enumerate(engine, name):
    """Enumerate through the GJ warp kernel (k_last_gj_warp<ENUM>): the bag of
    output tuples equals the oracle's, and the same pass folds count/checksum."""
    w = {"triangle": lambda: configs.triangle(scale=12, m=40000, seed=6),
         "clique4": lambda: configs.clique4(scale=11, m=30000)}[name]()
    q, plan, rels = fjg.prepare_workload(engine, w)
    rows, r = q.enumerate()
    ref = oracle.execute(w.query, plan, w.atom_columns(), output_mode="enumerate")
    assert r.count == len(rows) == ref["count"] and r.checksum == ref["checksum"]
    assert bag_equal(rows, ref["tuples"])
