"""Ingestion and fixture generators."""
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2301_10841_b200 import IoError, ParseError, ValidationError, fixtures, plan as P


def test_csv_round_trip_and_errors(tmp_path):
    cols = [np.array([1, -2, 2**31 - 1], np.int32), np.array([0, 5, -2**31], np.int32)]
    p = str(tmp_path / "r.csv")
    fixtures.write_csv(p, cols)
    got = fixtures.load_csv(p, 2)
    assert all((g == c).all() for g, c in zip(got, cols))
    (tmp_path / "empty.csv").write_text("")
    assert len(fixtures.load_csv(str(tmp_path / "empty.csv"), 2)[0]) == 0
    (tmp_path / "bad.csv").write_text("1,2\n3,x\n")
    with pytest.raises(ParseError, match="row 1 column 1"):
        fixtures.load_csv(str(tmp_path / "bad.csv"), 2)
    (tmp_path / "arity.csv").write_text("1,2\n3\n")
    with pytest.raises(ValidationError):
        fixtures.load_csv(str(tmp_path / "arity.csv"), 2)
    (tmp_path / "q.csv").write_text('1,"2"\n')
    with pytest.raises(ParseError):
        fixtures.load_csv(str(tmp_path / "q.csv"), 2)
    with pytest.raises(IoError):
        fixtures.load_csv(str(tmp_path / "missing.csv"), 2)


def test_gen_clover(tmp_path):
    fixtures.gen_clover(2, str(tmp_path))
    q, rels = fixtures.load_fixture(str(tmp_path))
    assert all(len(c[0]) == 5 for _, c in rels.values())          # 2n+1 rows
    cols = [rels[a["rel"]][1] for a in q["query"]]
    truth = oracle.brute_force(q, cols)
    assert truth.tolist() == [[0, 100, 200, 300]]                   # (x0, a0, b0, c0)
    for mode in ("binary", "free", "generic"):
        plan = P.compile_plan(q, mode)
        assert oracle.execute(q, plan, cols)["count"] == 1


def test_gen_random_deterministic(tmp_path):
    spec = {"atoms": 3, "arities": [2, 2, 1], "rows": 40, "domain": 5, "skew": 2.0}
    fixtures.gen_random(spec, 7, str(tmp_path / "a"))
    fixtures.gen_random(spec, 7, str(tmp_path / "b"))
    for f in os.listdir(tmp_path / "a"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()
    one = {"atoms": 2, "arities": [1, 1], "rows": 6, "domain": 1, "vars": 2}
    fixtures.gen_random(one, 1, str(tmp_path / "c"))
    q, rels = fixtures.load_fixture(str(tmp_path / "c"))
    cols = [rels[a["rel"]][1] for a in q["query"]]
    if q["query"][0]["vars"] != q["query"][1]["vars"]:             # domain 1: full Cartesian product
        assert len(oracle.brute_force(q, cols)) == 36


@pytest.mark.gpu
def test_fixture_on_device(engine, tmp_path):
    fixtures.gen_clover(50, str(tmp_path))
    q, rels = fixtures.load_fixture(str(tmp_path))
    dev = {n: engine.relation(c) for n, (_, c) in rels.items()}
    for mode in ("binary", "free", "generic"):
        plan = P.compile_plan(q, mode)
        r = engine.query({"query": q["query"]}, plan, [dev[a["rel"]] for a in q["query"]]).execute()
        assert r.count == 1
