"""Bushy binary plans: run_segments (PAPER §2.2).

decompose_bushy splits the tree into dependency-ordered left-deep segments;
every non-final segment is compiled (binary2fj, then factor / fj_to_gj by
mode), executed in enumerate mode on the device, and its output materialised
as a device-resident relation (fjg_query_output_relation) whose schema is all
variables of the segment ("materialized intermediates carry all base-table
attributes"); the parent segment uses it as an ordinary atom. The
final segment runs with the original query's head order, so its checksum is
the one the un-decomposed query would produce.
"""
from . import plan as P
from .configs import left_deep


def head_order(atoms):
    out = []
    for a in atoms:
        for v in a["vars"]:
            if v not in out:
                out.append(v)
    return out


def run_segments(engine, query, tree, relations, mode="free", output_mode="count", **exec_kw):
    """query: list of atoms; tree: binary plan ("R" | ["join", l, r]);
    relations: atom name -> device Relation. Returns (final ExecResult,
    final Query, [per-segment (name, plan, ExecResult)])."""
    atoms = {a["rel"]: a for a in query}
    head = head_order(query)
    segs = P.decompose_bushy(tree, query)
    inter = {}
    trace = []
    for idx, seg in enumerate(segs):
        name = f"P{idx + 1}"
        seg_atoms = [atoms[n] if n in atoms else inter[n][0] for n in seg]
        seg_vars = [v for v in head if any(v in a["vars"] for a in seg_atoms)]
        plan = P.compile_plan({"query": seg_atoms, "binary_plan": left_deep(seg)}, mode)
        rels = [relations[n] if n in atoms else inter[n][1] for n in seg]
        q = engine.query({"query": seg_atoms, "head": seg_vars}, plan, rels)
        if idx == len(segs) - 1:
            if output_mode == "enumerate":
                rows, r = q.enumerate(**exec_kw)
                r.extra["rows"] = rows
            else:
                r = q.execute(output_mode=output_mode, **exec_kw)
            trace.append((name, plan, r))
            return r, q, trace
        rows, r = q.enumerate(**exec_kw)
        inter[name] = ({"rel": name, "vars": seg_vars}, q.output_relation())
        trace.append((name, plan, r))
        q.close()
