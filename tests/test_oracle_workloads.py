"""The oracle-side restatement of the configs (oracle/workloads.py, inputs from
oracle/gen.cpp, plans from oracle/workload_plans.json) equals the product's
configs (paper_2301_10841_b200/configs.py, libfjgen.so, host plan compiler):
same queries, filters, aggregates, parameters, input bytes and plans. This is
what lets `bench.py --impl reference` run without any product library."""
import numpy as np
import pytest

from oracle import gen, workloads as OW
from paper_2301_10841_b200 import configs, datagen, plan as P

SMALL = {"chain": dict(n=5000, domain=3000), "triangle": dict(scale=12, m=30000),
         "star": dict(nf=20000, dims=(500, 400, 300, 200)), "clique4": dict(scale=12, m=30000),
         "path5": dict(scale=10, m=8000), "scale_triangle": dict(scale=11, m=9000),
         "scale_path5": dict(scale=11, m=9000)}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_workload_matches_product(name):
    kw = SMALL[name]
    a = OW.CONFIGS[name](**kw)
    b = configs.CONFIGS[name](**kw)
    assert a.name == b.name and a.query == b.query and a.atom_rel == b.atom_rel and a.mode == b.mode
    assert a.params == b.params and a.min_var == b.min_var and a.output_mode == b.output_mode
    assert {k: [tuple(p) for p in v] for k, v in a.filters.items()} == \
        {k: [tuple(p) for p in v] for k, v in b.filters.items()}
    assert sorted(a.relations) == sorted(b.relations)
    for r in a.relations:
        assert len(a.relations[r]) == len(b.relations[r])
        for x, y in zip(a.relations[r], b.relations[r]):
            assert x.dtype == np.int32 and (x == y).all()
    compiled = P.compile_plan({"query": b.query, "binary_plan": b.binary_plan}, b.mode)
    assert a.plan == [[[r, list(vs)] for (r, vs) in node] for node in compiled]
    assert a.input_tuples() == b.input_tuples()
    assert a.head() == P.head_variables(b.query)
    for x, y in zip(a.atom_columns(), b.atom_columns()):
        assert all((u == v).all() for u, v in zip(x, y))


def test_generators_full_size_c2():
    """C2's full-size R-MAT (2^20 vertices, 4M edges) is byte-identical."""
    a = gen.rmat(42, 20, 4 << 20)
    b = datagen.rmat(42, 20, 4 << 20)
    assert all((x == y).all() for x, y in zip(a, b))


def test_generators_edge_cases():
    assert len(gen.rmat(1, 3, 0)[0]) == 0
    s, d = gen.rmat(9, 4, 200)  # 200 of at most 240 distinct non-loop edges on 16 vertices: K grows
    bs, bd = datagen.rmat(9, 4, 200)
    assert (s == bs).all() and (d == bd).all()
    assert len(set(zip(s.tolist(), d.tolist()))) == 200 and not (s == d).any()
    assert (gen.zipf(3, 1, 1000, 1, 1.1) == 0).all()
