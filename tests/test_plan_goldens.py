"""Plan compiler goldens: the worked examples of SPEC.md:129-240 (SPEC acceptance
#3) through the host C++ compiler behind the C-ABI."""
import pytest

from paper_2301_10841_b200 import ValidationError, plan as P

CLOVER = [{"rel": "R", "vars": ["x", "a"]}, {"rel": "S", "vars": ["x", "b"]}, {"rel": "T", "vars": ["x", "c"]}]
EQ2 = [[("R", ["x", "a"]), ("S", ["x"])], [("S", ["b"]), ("T", ["x"])], [("T", ["c"])]]
EQ2_FACTORED = [[("R", ["x", "a"]), ("S", ["x"]), ("T", ["x"])], [("S", ["b"])], [("T", ["c"])]]
EQ3 = [[("R", ["x"]), ("S", ["x"]), ("T", ["x"])], [("R", ["a"])], [("S", ["b"])], [("T", ["c"])]]
CHAIN4 = [{"rel": "R", "vars": ["x", "y"]}, {"rel": "S", "vars": ["y", "z"]}, {"rel": "T", "vars": ["z", "u"]},
          {"rel": "W", "vars": ["u", "v"]}]
TRI = [{"rel": "R", "vars": ["x", "y"]}, {"rel": "S", "vars": ["y", "z"]}, {"rel": "T", "vars": ["x", "z"]}]
TRI_FACTORED = [[("R", ["x", "y"]), ("S", ["y"]), ("T", ["x"])], [("S", ["z"]), ("T", ["z"])]]


def test_binary2fj_clover_eq2():
    plan, warnings = P.binary2fj(["R", "S", "T"], CLOVER)
    assert plan == EQ2
    assert warnings == []


def test_binary2fj_chain():
    plan, _ = P.binary2fj(["R", "S", "T", "W"], CHAIN4)
    assert plan == [[("R", ["x", "y"]), ("S", ["y"])], [("S", ["z"]), ("T", ["z"])], [("T", ["u"]), ("W", ["u"])],
                    [("W", ["v"])]]


def test_binary2fj_singleton():
    plan, _ = P.binary2fj(["R"], CLOVER)
    assert plan == [[("R", ["x", "a"])]]


def test_binary2fj_cartesian_warns():
    q = [{"rel": "R", "vars": ["x"]}, {"rel": "S", "vars": ["y"]}]
    plan, warnings = P.binary2fj(["R", "S"], q)
    assert plan == [[("R", ["x"]), ("S", [])], [("S", ["y"])]]
    assert warnings and "cartesian" in warnings[0]


def test_factor_eq2():
    assert P.factor(EQ2, CLOVER) == EQ2_FACTORED


def test_factor_idempotent():
    assert P.factor(EQ2_FACTORED, CLOVER) == EQ2_FACTORED


def test_factor_chain_noop():
    plan, _ = P.binary2fj(["R", "S", "T", "W"], CHAIN4)
    assert P.factor(plan, CHAIN4) == plan


def test_schemas_eq2():
    assert P.derive_ght_schemas(EQ2, CLOVER) == {"R": [["x", "a"]], "S": [["x"], ["b"]], "T": [["x"], ["c"]]}


def test_schemas_triangle():  # SPEC.md:230, Example 3.8
    assert P.derive_ght_schemas(TRI_FACTORED, TRI) == {"R": [["x", "y"]], "S": [["y"], ["z"]],
                                                       "T": [["x"], ["z"], []]}


def test_schemas_single():
    assert P.derive_ght_schemas([[("R", ["x", "a"])]], CLOVER[:1]) == {"R": [["x", "a"]]}


def test_fj_to_gj_clover_eq3():
    assert P.fj_to_gj_plan(EQ2_FACTORED, CLOVER) == EQ3
    assert P.gj_variable_order(EQ2_FACTORED, CLOVER) == ["x", "a", "b", "c"]


def test_fj_to_gj_single():
    assert P.fj_to_gj_plan([[("R", ["x", "a"])]], CLOVER[:1]) == [[("R", ["x"])], [("R", ["a"])]]


def test_fj_to_gj_triangle():
    assert P.fj_to_gj_plan(TRI_FACTORED, TRI) == [[("R", ["x"]), ("T", ["x"])], [("R", ["y"]), ("S", ["y"])],
                                                 [("S", ["z"]), ("T", ["z"])]]


def test_vs_avs_covers():
    assert P.vs(EQ2, CLOVER, 0) == {"x", "a"}
    assert P.vs(EQ2, CLOVER, 1) == {"b", "x"}
    assert P.avs(EQ2, CLOVER, 1) == {"x", "a"}
    assert P.avs(EQ2, CLOVER, 0) == set()
    assert P.avs(EQ3, CLOVER, 3) == {"x", "a", "b"}
    assert P.covers(EQ2, CLOVER, 0) == [0]
    assert P.covers(EQ3, CLOVER, 0) == [0, 1, 2]
    assert P.covers(EQ2, CLOVER, 2) == [0]


def test_validate():
    assert P.validate(EQ2, CLOVER) == ""
    bad = [[("R", ["x", "a"]), ("S", ["x", "b"]), ("T", ["x", "c"])]]  # Example 3.7
    assert "no cover" in P.validate(bad, CLOVER)
    missing = [[("R", ["x", "a"]), ("S", ["x"])], [("S", ["b"]), ("T", ["x"])]]
    assert "partitioning" in P.validate(missing, CLOVER)
    dup = [[("R", ["x", "a"]), ("R", ["x"])]]
    assert "twice" in P.validate(dup, CLOVER)


def test_decompose_bushy():  # SPEC.md:201-203, acceptance #7
    q = [{"rel": n, "vars": [n.lower()]} for n in "RSTUABCDEF"]
    assert P.decompose_bushy(["join", ["join", "R", "S"], ["join", "T", "U"]], q) == [["T", "U"], ["R", "S", "P1"]]
    assert P.decompose_bushy(["join", ["join", "R", "S"], "T"], q) == [["R", "S", "T"]]
    segs = P.decompose_bushy(["join", ["join", ["join", "A", "B"], ["join", "C", "D"]], ["join", "E", "F"]], q)
    assert segs == [["C", "D"], ["E", "F"], ["A", "B", "P1", "P2"]]


def test_compile_modes():
    assert P.compile_plan(CLOVER, "binary") == EQ2
    assert P.compile_plan(CLOVER, "free") == EQ2_FACTORED
    assert P.compile_plan(CLOVER, "generic") == EQ3


def test_compile_rejects_bushy_and_duplicates():
    q = {"query": CHAIN4, "binary_plan": ["join", ["join", "R", "S"], ["join", "T", "W"]]}
    with pytest.raises(ValidationError):
        P.compile_plan(q, "free")
    with pytest.raises(ValidationError):
        P.compile_plan([{"rel": "R", "vars": ["x"]}, {"rel": "R", "vars": ["y"]}], "free")


def test_config_plans():
    """The five BASELINE configs compile to the plans SURVEY.md §8(a) derives."""
    from paper_2301_10841_b200 import configs
    w = configs.chain(n=100, domain=100)
    assert P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode) == [
        [("R", ["a", "b"]), ("S", ["b"])], [("S", ["c"]), ("T", ["c"])], [("T", ["d"])]]
    w = configs.triangle(scale=8, m=500)
    assert P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode) == [
        [("E1", ["a"]), ("E3", ["a"])], [("E1", ["b"]), ("E2", ["b"])], [("E2", ["c"]), ("E3", ["c"])]]
    w = configs.star(nf=1000, dims=(100, 80, 30, 10))
    assert P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode) == [
        [("F", ["r", "f1", "f2", "f3", "f4"]), ("D1", ["f1"]), ("D2", ["f2"]), ("D3", ["f3"]), ("D4", ["f4"])],
        [("D1", ["x1"])], [("D2", ["x2"])], [("D3", ["x3"])], [("D4", ["x4"])]]
    w = configs.clique4(scale=8, m=1000)
    assert P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode) == [
        [("Eab", ["a"]), ("Eac", ["a"]), ("Ead", ["a"])], [("Eab", ["b"]), ("Ebc", ["b"]), ("Ebd", ["b"])],
        [("Eac", ["c"]), ("Ebc", ["c"]), ("Ecd", ["c"])], [("Ead", ["d"]), ("Ebd", ["d"]), ("Ecd", ["d"])]]
