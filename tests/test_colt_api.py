"""The GHT / COLT handle at the C-ABI (fjg_colt_*; Fig 5,
SPEC.md:286-339): new is free (BaseScan), force is lazy and idempotent, get /
iter / rows / estimated_key_count agree with a numpy model of the trie, and
the state persists across calls. Symbols are checked on the CPU by
tests/test_capi.py; these tests need the GPU."""
import numpy as np
import pytest

import paper_2301_10841_b200 as fjg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    e = fjg.Engine(0)
    yield e
    e.close()


def model(cols, keycols):
    """key tuple -> sorted list of row indices"""
    out = {}
    for i in range(len(cols[0])):
        out.setdefault(tuple(int(cols[c][i]) for c in keycols), []).append(i)
    return out


def test_colt_two_levels(engine):
    rng = np.random.default_rng(5)
    n = 5000
    x = rng.integers(0, 300, n).astype(np.int32)
    y = rng.integers(-50, 50, n).astype(np.int32)
    z = rng.integers(0, 10**6, n).astype(np.int32)
    rel = engine.relation([x, y, z])
    c = engine.colt(rel, [[0], [1]])  # vector level: column 2
    assert c.nlevels == 3
    # GHT new does no work: the root is a BaseScan of n rows
    assert c.estimated_key_count(0) == n
    keys0 = c.iter(0)
    m0 = model([x, y, z], [0])
    assert sorted(k for k, _ in keys0) == sorted(m0)
    assert c.estimated_key_count(0) == len(m0)  # forced map: its keys
    assert sum(ln for _, (_, ln) in keys0) == n
    for (k, sub) in keys0[:50]:
        assert sub[1] == len(m0[k])
        # level 1 unforced: estimated count = its length
        assert c.estimated_key_count(1, sub) == sub[1]
        kids = c.iter(1, sub)
        m1 = model([x[m0[k]], y[m0[k]]], [1])
        assert sorted(kk for kk, _ in kids) == sorted(m1)
        assert c.estimated_key_count(1, sub) == len(m1)
        for (kk, ch) in kids:
            rows_z = sorted(c.rows(2, ch, 2).tolist())
            assert rows_z == sorted(z[[m0[k][i] for i in m1[kk]]].tolist())
    # batched get, with misses, on the root and on level-1 subtries
    probe = [(int(v),) for v in rng.integers(-5, 310, 400)]
    got = c.get(0, [(0, n)] * len(probe), probe)
    by_key = dict(keys0)
    for kv, g in zip(probe, got):
        assert (g is None) == (kv not in m0)
        if g is not None:
            assert g == by_key[kv]
    k, sub = keys0[0]
    ys = [(int(v),) for v in range(-60, 60)]
    got = c.get(1, [sub] * len(ys), ys)
    m1 = model([x[m0[k]], y[m0[k]]], [1])
    assert [g is not None for g in got] == [kv in m1 for kv in ys]
    # idempotent force, state persists
    c.force(1, [sub, sub])
    assert c.iter(1, sub) == c.iter(1, sub)
    c.close()


def test_colt_arity2_key(engine):
    rng = np.random.default_rng(6)
    n = 3000
    a = rng.integers(0, 20, n).astype(np.int32)
    b = rng.integers(0, 20, n).astype(np.int32)
    rel = engine.relation([a, b])
    c = engine.colt(rel, [[0, 1]])
    m = model([a, b], [0, 1])
    keys = c.iter(0)
    assert sorted(k for k, _ in keys) == sorted(m)
    assert all(sub[1] == len(m[k]) for k, sub in keys)
    probe = [(int(u), int(v)) for u, v in rng.integers(0, 22, (300, 2))]
    got = c.get(0, [(0, n)] * len(probe), probe)
    assert [g is not None for g in got] == [p in m for p in probe]
    c.close()


def test_colt_empty_and_errors(engine):
    rel = engine.relation([np.zeros(0, np.int32), np.zeros(0, np.int32)])
    c = engine.colt(rel, [[0]])
    assert c.iter(0) == [] and c.estimated_key_count(0) == 0
    c.close()
    rel2 = engine.relation([np.arange(10, dtype=np.int32)])
    with pytest.raises(fjg.ValidationError):
        engine.colt(rel2, [[0], [0]])
    c2 = engine.colt(rel2, [[0]])
    with pytest.raises(fjg.ValidationError):
        c2.iter(3)
    c2.close()
