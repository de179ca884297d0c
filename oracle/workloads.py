"""ORACLE WORKLOADS — TEST / BASELINE INFRASTRUCTURE ONLY. The BASELINE.json
configs restated on the oracle side (queries, filters, aggregates, inputs from
oracle/gen.py, Free Join plans from oracle/workload_plans.json), so that
`bench.py --impl reference` runs the CPU restatement of the reference path
without importing or loading anything from the product package.
tests/test_oracle_workloads.py checks every field against the product's
paper_2301_10841_b200/configs.py and plan compiler.
"""
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import gen

M = 1 << 20
_PLANS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "workload_plans.json")


@dataclass
class OWorkload:
    name: str
    query: list
    atom_rel: list
    relations: dict
    filters: dict = field(default_factory=dict)
    min_var: str = None
    params: dict = field(default_factory=dict)
    output_mode: str = "count"
    plan_key: str = ""
    mode: str = "free"  # plan mode the plan was compiled in (binary | free | generic)
    plan_override: list = None

    @property
    def plan(self):
        if self.plan_override is not None:
            return self.plan_override
        with open(_PLANS) as f:
            return json.load(f)[self.plan_key or self.name]

    def filtered(self):
        out = {}
        ops = {"<": np.less, "<=": np.less_equal, ">": np.greater, ">=": np.greater_equal, "=": np.equal,
               "!=": np.not_equal}
        for name, cols in self.relations.items():
            keep = np.ones(len(cols[0]), dtype=bool)
            for (c, op, k) in self.filters.get(name, []):
                keep &= ops[op](cols[c].astype(np.int64), k)
            out[name] = cols if not self.filters.get(name) else [c[keep] for c in cols]
        return out

    def atom_columns(self):
        rels = self.filtered()
        return [rels[r] for r in self.atom_rel]

    def input_tuples(self):
        return int(sum(len(self.relations[r][0]) for r in self.atom_rel))

    def head(self):
        seen = []
        for a in self.query:
            for v in a["vars"]:
                if v not in seen:
                    seen.append(v)
        return seen


def _edges(names_vars):
    return [{"rel": n, "vars": list(v)} for (n, v) in names_vars]


def chain(n=M, domain=1 << 20, seed=1):
    rels = {name: [gen.uniform(seed + i, 0, n, domain), gen.uniform(seed + i, 1, n, domain)]
            for i, name in enumerate("RST")}
    q = _edges([("R", "ab"), ("S", "bc"), ("T", "cd")])
    return OWorkload("chain", q, ["R", "S", "T"], rels, params={"rows": n, "domain": domain, "seed": seed})


def triangle(scale=20, m=4 * M, seed=42, name="triangle"):
    q = _edges([("E1", "ab"), ("E2", "bc"), ("E3", "ac")])
    return OWorkload(name, q, ["E"] * 3, {"E": gen.rmat(seed, scale, m)},
                     params={"scale": scale, "edges": m, "seed": seed}, plan_key="triangle", mode="generic")


def star(nf=32 * M, dims=(int(2.5 * M), 4 * M, 1 * M, 100_000), thresh=(100, 50, 20, 10), s=1.1, seed=7):
    rels = {"F": [np.arange(nf, dtype=np.int32)] + [gen.zipf(seed, 10 + i, nf, n, s) for i, n in enumerate(dims)]}
    q = [{"rel": "F", "vars": ["r", "f1", "f2", "f3", "f4"]}]
    filters = {}
    for i, n in enumerate(dims):
        d = f"D{i + 1}"
        rels[d] = [np.arange(n, dtype=np.int32), gen.uniform(seed + 100 + i, 0, n, 1000)]
        filters[d] = [(1, "<", thresh[i])]
        q.append({"rel": d, "vars": [f"f{i + 1}", f"x{i + 1}"]})
    return OWorkload("star", q, ["F"] + [f"D{i + 1}" for i in range(len(dims))], rels, filters=filters, min_var="r",
                     params={"fact_rows": nf, "dims": list(dims), "thresholds": list(thresh), "zipf_s": s,
                             "seed": seed})


def clique4(scale=22, m=16 * M, seed=11):
    o = gen.orient(seed, *gen.rmat(seed, scale, m))
    atoms = [("Eab", "ab"), ("Eac", "ac"), ("Ebc", "bc"), ("Ead", "ad"), ("Ebd", "bd"), ("Ecd", "cd")]
    return OWorkload("clique4", _edges(atoms), ["E"] * 6, {"E": o},
                     params={"scale": scale, "generated_edges": m, "oriented_edges": int(len(o[0])), "seed": seed},
                     mode="generic")


def path5(scale=27, m=512 * M, seed=5, name="path5"):
    vs = "abcdef"
    q = _edges([(f"E{i + 1}", vs[i] + vs[i + 1]) for i in range(5)])
    return OWorkload(name, q, ["E"] * 5, {"E": gen.rmat(seed, scale, m)},
                     params={"scale": scale, "edges": m, "seed": seed}, output_mode="factorized_count",
                     plan_key="path5")


def scale_triangle(scale=27, m=512 * M, seed=5):
    return triangle(scale, m, seed, name="scale_triangle")


def scale_path5(scale=27, m=512 * M, seed=5):
    return path5(scale, m, seed, name="scale_path5")


CONFIGS = {"chain": chain, "triangle": triangle, "star": star, "clique4": clique4, "path5": path5,
           "scale_triangle": scale_triangle, "scale_path5": scale_path5}
