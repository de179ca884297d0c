"""The five BASELINE.json configurations as workloads (query, binary plan,
plan mode, seeded relations, filters, aggregate), parameterised by size so the
tests can run them small and the bench at full size.

Self-joins are renamed atoms bound to one relation.
"""
import json
from dataclasses import dataclass, field

import numpy as np

from . import datagen
from .datagen import M


@dataclass
class Workload:
    name: str
    query: list                      # [{"rel": atom name, "vars": [...]}, ...]
    binary_plan: object              # left-deep tree over atom names
    mode: str                        # binary | free | generic
    relations: dict                  # base relation name -> list of int32 columns
    atom_rel: list                   # base relation per atom
    filters: dict = field(default_factory=dict)  # base relation -> [(col, op, const)]
    min_var: str = None
    params: dict = field(default_factory=dict)
    output_mode: str = "count"     # factorized_count for the 5-path (memoised chain count)

    @property
    def query_json(self):
        return json.dumps({"query": self.query, "binary_plan": self.binary_plan})

    def filtered(self):
        """apply_filter on the host (oracle side; the device uses fjg_relation_filter)."""
        out = {}
        for name, cols in self.relations.items():
            preds = self.filters.get(name, [])
            if not preds:
                out[name] = cols
                continue
            keep = np.ones(len(cols[0]), dtype=bool)
            for (c, op, k) in preds:
                x = cols[c].astype(np.int64)
                keep &= {"<": x < k, "<=": x <= k, ">": x > k, ">=": x >= k, "=": x == k, "!=": x != k}[op]
            out[name] = [c[keep] for c in cols]
        return out

    def atom_columns(self, filtered=True):
        rels = self.filtered() if filtered else self.relations
        return [rels[r] for r in self.atom_rel]

    def input_tuples(self):
        """Σ over atoms of relation rows, pre-filter."""
        return int(sum(len(self.relations[r][0]) for r in self.atom_rel))


def left_deep(names):
    t = names[0]
    for n in names[1:]:
        t = ["join", t, n]
    return t


def chain(n=M, domain=1 << 20, seed=1):
    """C1: Q(a,b,c,d) :- R(a,b),S(b,c),T(c,d); 1M rows x 2 int32, U[0,2^20)."""
    rels = {}
    for i, name in enumerate("RST"):
        s = seed + i
        rels[name] = [datagen.uniform(s, 0, n, domain), datagen.uniform(s, 1, n, domain)]
    q = [{"rel": "R", "vars": ["a", "b"]}, {"rel": "S", "vars": ["b", "c"]}, {"rel": "T", "vars": ["c", "d"]}]
    return Workload("chain", q, left_deep(["R", "S", "T"]), "free", rels, ["R", "S", "T"],
                    params={"rows": n, "domain": domain, "seed": seed})


def triangle(scale=20, m=4 * M, seed=42):
    """C2: Q(a,b,c) :- E(a,b),E(b,c),E(a,c) on R-MAT(.57,.19,.19,.05); GJ order a,b,c."""
    src, dst = datagen.rmat(seed, scale, m)
    q = [{"rel": "E1", "vars": ["a", "b"]}, {"rel": "E2", "vars": ["b", "c"]}, {"rel": "E3", "vars": ["a", "c"]}]
    return Workload("triangle", q, left_deep(["E1", "E2", "E3"]), "generic", {"E": [src, dst]}, ["E", "E", "E"],
                    params={"scale": scale, "edges": m, "seed": seed})


STAR_DIMS = (int(2.5 * M), 4 * M, 1 * M, 100_000)
STAR_THRESH = (100, 50, 20, 10)  # attr ~ U[0,1000): 10% / 5% / 2% / 1%


def star(nf=32 * M, dims=STAR_DIMS, thresh=STAR_THRESH, s=1.1, seed=7):
    """C3: F(r,f1..f4) with Zipf(1.1) FKs into D1..D4(fi, xi), Di filtered xi < t_i;
    factorised left-deep plan; COUNT + MIN(F.rowid) + checksum."""
    fcols = [np.arange(nf, dtype=np.int32)]
    for i, n in enumerate(dims):
        fcols.append(datagen.zipf(seed, 10 + i, nf, n, s))
    rels = {"F": fcols}
    filters = {}
    q = [{"rel": "F", "vars": ["r", "f1", "f2", "f3", "f4"]}]
    for i, n in enumerate(dims):
        name = f"D{i + 1}"
        rels[name] = [np.arange(n, dtype=np.int32), datagen.uniform(seed + 100 + i, 0, n, 1000)]
        filters[name] = [(1, "<", thresh[i])]
        q.append({"rel": name, "vars": [f"f{i + 1}", f"x{i + 1}"]})
    names = ["F"] + [f"D{i + 1}" for i in range(len(dims))]
    return Workload("star", q, left_deep(names), "free", rels, names, filters=filters, min_var="r",
                    params={"fact_rows": nf, "dims": list(dims), "thresholds": list(thresh), "zipf_s": s,
                            "seed": seed})


def clique4(scale=22, m=16 * M, seed=11):
    """C4: 4-clique over the 6 edge atoms of an R-MAT graph oriented by (degree, id); GJ a,b,c,d."""
    src, dst = datagen.rmat(seed, scale, m)
    osrc, odst = datagen.orient(seed, src, dst)
    atoms = [("Eab", "a", "b"), ("Eac", "a", "c"), ("Ebc", "b", "c"), ("Ead", "a", "d"), ("Ebd", "b", "d"),
             ("Ecd", "c", "d")]
    q = [{"rel": n, "vars": [x, y]} for (n, x, y) in atoms]
    return Workload("clique4", q, left_deep([a[0] for a in atoms]), "generic", {"E": [osrc, odst]}, ["E"] * 6,
                    params={"scale": scale, "generated_edges": m, "oriented_edges": int(len(osrc)),
                            "seed": seed})


def path5(scale=27, m=512 * M, seed=5):
    """C5 5-way path Q :- E(a,b),E(b,c),E(c,d),E(d,e),E(e,f) (count only)."""
    src, dst = datagen.rmat(seed, scale, m)
    vs = "abcdef"
    q = [{"rel": f"E{i + 1}", "vars": [vs[i], vs[i + 1]]} for i in range(5)]
    return Workload("path5", q, left_deep([f"E{i + 1}" for i in range(5)]), "free", {"E": [src, dst]}, ["E"] * 5,
                    params={"scale": scale, "edges": m, "seed": seed}, output_mode="factorized_count")


def scale_triangle(scale=27, m=512 * M, seed=5):
    """C5 triangle at R-MAT 2^27 / 512M edges."""
    w = triangle(scale, m, seed)
    w.name = "scale_triangle"
    return w


def scale_path5(scale=27, m=512 * M, seed=5):
    """C5 5-path at R-MAT 2^27 / 512M edges (count only, memoised)."""
    w = path5(scale, m, seed)
    w.name = "scale_path5"
    return w


CONFIGS = {"scale_path5": scale_path5, "chain": chain, "triangle": triangle, "star": star, "clique4": clique4, "path5": path5,
           "scale_triangle": scale_triangle}
