"""Python mirror of the reference's query-ir and plan-compiler operations.

Every function calls the host C++ plan compiler through the C-ABI
(fjg_plan_op / fjg_compile_plan); names and argument meaning follow
SPEC.md:129-240. Plans are lists of nodes, nodes lists of (relation, [vars])
subatoms; queries are lists of {"rel": name, "vars": [...]} atoms.
"""
import json

from . import _capi

BINARY, FREE, GENERIC = 0, 1, 2
_MODES = {"binary": BINARY, "free": FREE, "generic": GENERIC}


def _q(query):
    if isinstance(query, str):
        return query
    if isinstance(query, dict):
        return json.dumps(query)
    return json.dumps({"query": query})


def _plan_obj(plan):
    return [[[r, list(v)] for (r, v) in node] for node in plan]


def _load_plan(s):
    return [[(r, list(v)) for (r, v) in node] for node in json.loads(s)]


def _op(op, query, arg):
    return _capi.call_str(_capi.lib.fjg_plan_op, op.encode(), _q(query).encode(), json.dumps(arg).encode())


def compile_plan(query, mode="free", binary_plan=None, factor_fixpoint=False):
    """decompose -> binary2fj -> (factor if free) -> (fj_to_gj if generic) -> validate."""
    if isinstance(mode, str):
        mode = _MODES[mode]
    q = query
    if not isinstance(q, (str, dict)):
        q = {"query": q}
    if isinstance(q, dict) and binary_plan is not None:
        q = dict(q, binary_plan=binary_plan)
    s = _capi.call_str(_capi.lib.fjg_compile_plan, _q(q).encode(), int(mode), int(bool(factor_fixpoint)))
    return _load_plan(s)


def binary2fj(segment, query):
    """Fig 9. Returns (plan, warnings)."""
    r = json.loads(_op("binary2fj", query, list(segment)))
    return _load_plan(json.dumps(r["plan"])), r["warnings"]


def factor(plan, query, fixpoint=False):
    """Fig 10."""
    return _load_plan(_op("factor_fixpoint" if fixpoint else "factor", query, _plan_obj(plan)))


def fj_to_gj_plan(plan, query):
    """SPEC.md:232-240."""
    return _load_plan(_op("fj_to_gj", query, _plan_obj(plan)))


def gj_variable_order(plan, query):
    return json.loads(_op("gj_order", query, _plan_obj(plan)))


def derive_ght_schemas(plan, query):
    """{relation: [[vars], ...]} (a trailing [] is the leaf vector)."""
    return json.loads(_op("schemas", query, _plan_obj(plan)))


def validate(plan, query):
    """'' if valid, else the first violation with its node index."""
    return json.loads(_op("validate", query, _plan_obj(plan)))


def covers(plan, query, k):
    return json.loads(_op("covers", query, {"plan": _plan_obj(plan), "k": k}))


def vs(plan, query, k):
    return set(json.loads(_op("vs", query, {"plan": _plan_obj(plan), "k": k})))


def avs(plan, query, k):
    return set(json.loads(_op("avs", query, {"plan": _plan_obj(plan), "k": k})))


def decompose_bushy(tree, query):
    """dependency-ordered left-deep segments; intermediates are P1, P2, ..."""
    return json.loads(_op("decompose", query, tree))


def head_variables(query):
    return json.loads(_op("head_vars", query, None))


def plan_json(plan):
    return json.dumps(_plan_obj(plan))
