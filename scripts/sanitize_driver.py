"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every config at a tiny size, count + enumerate + the
SLT / SIMPLE backends + the memoised chain count + the multi-GPU path at world
1, each checked against the oracle. Used by scripts/sanitize.sh."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2301_10841_b200 as fjg  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2301_10841_b200 import configs, dist as D, plan as P  # noqa: E402
from randq import bag_equal  # noqa: E402

SMALL = {"chain": dict(n=3000, domain=3000), "triangle": dict(scale=10, m=6000, seed=3),
         "star": dict(nf=30000, dims=(500, 400, 300, 100)), "clique4": dict(scale=9, m=3000),
         "path5": dict(scale=9, m=3000)}


def main():
    eng = fjg.Engine(0)
    fails = 0
    for name, kw in SMALL.items():
        w = configs.CONFIGS[name](**kw)
        plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
        head = P.head_variables(w.query)
        mv = head.index(w.min_var) if w.min_var else -1
        ref = oracle.execute(w.query, plan, w.atom_columns(), min_var=mv, output_mode=w.output_mode)
        q, _, rels = fjg.prepare_workload(eng, w)
        for backend in ("colt", "slt", "simple"):
            for batch in (0, 7):
                r = q.execute(min_var=w.min_var, output_mode=w.output_mode, backend=backend, batch_size=batch)
                ok = r.count == ref["count"] and (w.output_mode != "count" or r.checksum == ref["checksum"])
                fails += not ok
                print(name, backend, batch, "ok" if ok else "MISMATCH", flush=True)
        if w.output_mode == "count":
            rows, r = q.enumerate()
            e = oracle.execute(w.query, plan, w.atom_columns(), output_mode="enumerate")
            ok = bag_equal(rows, e["tuples"])
            fails += not ok
            print(name, "enumerate", "ok" if ok else "MISMATCH", flush=True)
        q.close()
        comm = D.Comm(eng, 1, 0)
        sq = D.ShardedQuery(eng, w, plan, comm)
        r = sq.execute(min_var=w.min_var, output_mode=w.output_mode)
        ok = r.count == ref["count"]
        fails += not ok
        print(name, "multi(world 1)", "ok" if ok else "MISMATCH", flush=True)
        sq.close()
        comm.close()
    eng.close()
    print("FAILS", fails)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
