"""B200-native Free Join executor (arXiv 2301.10841): COLT build + vectorised
Free Join node execution as sm_100a kernels behind a C-ABI (include/fjg.h).

Host side (this package) mirrors the reference's interfaces: plan compiler
(plan.py -> host C++), relations / queries / execution (engine.py -> device),
multi-GPU sharding on the first plan variable (dist.py)."""
from . import fixtures, plan
from ._capi import EngineError, Error, IoError, ParseError, ResourceError, ValidationError
from .engine import Engine, ExecResult, Query, Relation

__all__ = ["plan", "Engine", "Relation", "Query", "ExecResult", "Error", "IoError", "ParseError",
           "ValidationError", "ResourceError", "EngineError", "run_workload", "prepare_workload"]


def prepare_workload(engine, w, device_relations=None):
    """Upload + filter the workload's relations, compile its plan on the host,
    bind one relation per atom. Returns (Query, plan, base relations)."""
    from . import plan as P
    rels = device_relations
    if rels is None:
        rels = {}
        for name, cols in w.relations.items():
            r = engine.relation(cols)
            if w.filters.get(name):
                r = r.filter(w.filters[name])
            rels[name] = r
    fj_plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    q = engine.query({"query": w.query}, fj_plan, [rels[r] for r in w.atom_rel])
    return q, fj_plan, rels


def run_workload(engine, w, **exec_kw):
    q, fj_plan, rels = prepare_workload(engine, w)
    kw = dict(exec_kw)
    if w.min_var is not None and "min_var" not in kw:
        kw["min_var"] = w.min_var
    if getattr(w, "output_mode", "count") != "count" and "output_mode" not in kw:
        kw["output_mode"] = w.output_mode
    return q.execute(**kw), q, fj_plan, rels
