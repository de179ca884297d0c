"""Seeded generators: determinism and the structural properties the configs
promise."""
import numpy as np

from paper_2301_10841_b200 import configs, datagen


def test_uniform_deterministic():
    a = datagen.uniform(1, 0, 10000, 1 << 20)
    b = datagen.uniform(1, 0, 10000, 1 << 20)
    c = datagen.uniform(1, 1, 10000, 1 << 20)
    assert (a == b).all() and not (a == c).all()
    assert a.min() >= 0 and a.max() < (1 << 20)


def test_rmat_properties():
    s, d = datagen.rmat(3, 12, 20000)
    assert len(s) == len(d) == 20000
    assert (s != d).all()
    keys = s.astype(np.int64) << 32 | d.astype(np.int64)
    assert len(np.unique(keys)) == 20000
    assert s.max() < (1 << 12) and d.max() < (1 << 12)
    # skew: vertex 0 region is the hub
    assert np.bincount(s).max() > 20 * np.bincount(s).mean()
    s2, d2 = datagen.rmat(3, 12, 20000)
    assert (s == s2).all() and (d == d2).all()
    # rows are in stream order, not sorted
    assert not (np.diff(s) >= 0).all()


def test_orient():
    s, d = datagen.rmat(4, 10, 5000)
    os_, od = datagen.orient(4, s, d)
    assert (os_ != od).all()
    und = np.unique(np.minimum(s, d).astype(np.int64) << 32 | np.maximum(s, d))
    assert len(os_) == len(und)
    deg = np.bincount(np.concatenate([os_, od]), minlength=1 << 10)
    rank_ok = (deg[os_] < deg[od]) | ((deg[os_] == deg[od]) & (os_ < od))
    assert rank_ok.all()


def test_zipf_range_and_skew():
    z = datagen.zipf(7, 10, 200000, 1000, 1.1)
    assert z.min() >= 0 and z.max() < 1000
    top = np.bincount(z).max() / len(z)
    assert 0.05 < top < 0.3


def test_config_shapes():
    w = configs.star(nf=5000, dims=(100, 200, 50, 10))
    assert len(w.relations["F"]) == 5 and len(w.relations["F"][0]) == 5000
    f = w.filtered()
    assert (f["D1"][1] < 100).all() and len(f["D1"][0]) < 100
    assert w.input_tuples() == 5000 + 100 + 200 + 50 + 10
    t = configs.triangle(scale=10, m=3000)
    assert t.atom_rel == ["E", "E", "E"] and t.input_tuples() == 9000
