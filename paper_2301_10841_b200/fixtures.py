"""Fixture I/O and generators (bench-cli module).

On-disk layout: <dir>/<relation>.csv (header-less, int
fields), <dir>/schema.txt (one line per relation: `name:attr1:int,attr2:int`,
SPEC.md:88) and <dir>/query.json (the plan-file dialect of SPEC.md:171).
CSV parsing is the host C++ `fjg_parse_csv`. Text columns (SPEC's Value::Text)
are not supported on the device; generators encode their constants as ints.
"""
import ctypes as C
import json
import os

import numpy as np

from . import _capi


def load_csv(path, ncols):
    """load_csv -> list of int32 columns, rows in file order."""
    rows = C.c_uint64(0)
    rc = _capi.lib.fjg_parse_csv(path.encode(), ncols, None, 0, C.byref(rows))
    if rc not in (_capi.FJG_OK, _capi.FJG_E_RESOURCE):
        _capi.check(rc)
    buf = np.empty((max(rows.value, 1), ncols), dtype=np.int32)
    _capi.check(_capi.lib.fjg_parse_csv(path.encode(), ncols, buf.ctypes.data, rows.value, C.byref(rows)))
    return [np.ascontiguousarray(buf[: rows.value, c]) for c in range(ncols)]


def write_csv(path, cols):
    n = len(cols[0]) if cols else 0
    with open(path, "w") as f:
        for i in range(n):
            f.write(",".join(str(int(c[i])) for c in cols) + "\n")


def write_fixture(out_dir, query, relations, binary_plan=None, extra=None):
    """relations: name -> (attribute names, columns)."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "schema.txt"), "w") as f:
        for name, (attrs, cols) in relations.items():
            f.write(name + ":" + ",".join(f"{a}:int" for a in attrs) + "\n")
            write_csv(os.path.join(out_dir, f"{name}.csv"), cols)
    q = {"query": query}
    if binary_plan is not None:
        q["binary_plan"] = binary_plan
    if extra:
        q.update(extra)
    with open(os.path.join(out_dir, "query.json"), "w") as f:
        json.dump(q, f)


def read_schema(path):
    out = {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            name, rest = line.split(":", 1)
            attrs = []
            for field in rest.split(","):
                attr, typ = field.rsplit(":", 1)
                if typ != "int":
                    raise _capi.ValidationError(f"{name}.{attr}: only int columns are supported on the device")
                attrs.append(attr)
            out[name] = attrs
    return out


def load_fixture(in_dir):
    """-> (query dict, {relation: (attrs, columns)})."""
    schema = read_schema(os.path.join(in_dir, "schema.txt"))
    rels = {name: (attrs, load_csv(os.path.join(in_dir, f"{name}.csv"), len(attrs))) for name, attrs in schema.items()}
    with open(os.path.join(in_dir, "query.json")) as f:
        q = json.load(f)
    return q, rels


# Fig 2 clover instance with ints for the constants:
# x_i -> i, a0/b0/c0 -> 100/200/300, a_i^l -> 1000+i, a_i^r -> 2000+i, ...
def clover_relations(n):
    R = [(0, 100)] + [(1, 1000 + i) for i in range(1, n + 1)] + [(2, 2000 + i) for i in range(1, n + 1)]
    S = [(0, 200)] + [(2, 3000 + i) for i in range(1, n + 1)] + [(3, 4000 + i) for i in range(1, n + 1)]
    T = [(0, 300)] + [(3, 5000 + i) for i in range(1, n + 1)] + [(1, 6000 + i) for i in range(1, n + 1)]
    cols = lambda rows: [np.array([r[0] for r in rows], np.int32), np.array([r[1] for r in rows], np.int32)]
    return {"R": (["x", "a"], cols(R)), "S": (["x", "b"], cols(S)), "T": (["x", "c"], cols(T))}


def gen_clover(n, out_dir):
    """gen_clover: the Fig 2 instance, 2n+1 rows per relation,
    query Q(x,a,b,c) :- R(x,a),S(x,b),T(x,c) with the binary plan [R,S,T]."""
    if n < 1:
        raise _capi.ValidationError("gen_clover: n must be >= 1")
    rels = clover_relations(n)
    query = [{"rel": k, "vars": v[0]} for k, v in rels.items()]
    write_fixture(out_dir, query, rels, binary_plan=["join", ["join", "R", "S"], "T"])


def gen_random(spec, seed, out_dir):
    """gen_random: spec = {"atoms": k, "arities": [..],
    "rows": r, "domain": d, "skew": s>=1}; deterministic in seed. Values are
    floor(d * u^skew) (skew > 1 piles mass on small keys: duplicated join
    keys). Atoms are named A0..; variables v0..v{d-1} drawn per atom."""
    rng = np.random.default_rng(seed)
    k = int(spec["atoms"])
    arities = spec.get("arities") or [2] * k
    nvars = int(spec.get("vars", max(arities) + 1))
    pool = [f"v{i}" for i in range(nvars)]
    rels, query = {}, []
    for a in range(k):
        vs = [str(x) for x in rng.choice(pool, size=arities[a], replace=False)]
        n = int(spec["rows"])
        cols = [np.floor(spec["domain"] * rng.random(n) ** spec.get("skew", 1.0)).astype(np.int32) for _ in vs]
        rels[f"A{a}"] = (vs, cols)
        query.append({"rel": f"A{a}", "vars": vs})
    tree = "A0"
    for a in range(1, k):
        tree = ["join", tree, f"A{a}"]
    write_fixture(out_dir, query, rels, binary_plan=tree, extra={"seed": seed, "spec": spec})
