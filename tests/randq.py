"""Seeded random (query, instance) generator for the property tests
(<=5 atoms, <=50 rows, small skewed domains with duplicates)."""
import numpy as np


def random_query(rng, max_atoms=5, max_rows=50):
    nvars = int(rng.integers(2, 6))
    pool = [f"v{i}" for i in range(nvars)]
    natoms = int(rng.integers(2, max_atoms + 1))
    atoms, cols = [], []
    domain = int(rng.integers(2, 7))
    for a in range(natoms):
        arity = int(rng.integers(1, min(3, nvars) + 1))
        vs = list(rng.choice(pool, size=arity, replace=False))
        atoms.append({"rel": f"A{a}", "vars": [str(v) for v in vs]})
        n = int(rng.integers(0 if rng.random() < 0.05 else 1, max_rows + 1))
        # skew: squaring a uniform pushes mass to small values; duplicates arise
        cs = [np.floor(domain * rng.random(n) ** 2).astype(np.int32) for _ in range(arity)]
        cols.append(cs)
    order = list(rng.permutation(natoms))
    tree = atoms[order[0]]["rel"]
    for i in order[1:]:
        tree = ["join", tree, atoms[i]["rel"]]
    return {"query": atoms, "binary_plan": tree}, cols


def sorted_rows(a):
    a = np.asarray(a, dtype=np.int64)
    if a.size == 0:
        return a.reshape(0, a.shape[1] if a.ndim == 2 else 0)
    return a[np.lexsort(a.T[::-1])]


def bag_equal(a, b):
    a, b = sorted_rows(a), sorted_rows(b)
    return a.shape == b.shape and bool((a == b).all())
