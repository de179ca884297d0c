"""Find random queries where an eager backend disagrees with the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import json
import numpy as np
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import plan as P
from oracle import oracle
from randq import random_query

eng = fjg.Engine(0)
rng = np.random.default_rng(4242)
bad = 0
for it in range(300):
    q, cols = random_query(rng)
    for mode in ("binary", "free", "generic"):
        plan = P.compile_plan(q, mode)
        ref = oracle.execute(q, plan, cols)
        rels = [eng.relation(c) for c in cols]
        qq = eng.query({"query": q["query"]}, plan, rels)
        out = {}
        for b in ("colt", "slt", "simple"):
            r1 = qq.execute(backend=b)
            r2 = qq.execute(backend=b)
            out[b] = (r1.count, r2.count)
        if any(v != (ref["count"], ref["count"]) for v in out.values()):
            bad += 1
            print("MISMATCH it", it, mode, "ref", ref["count"], out)
            print(" query", json.dumps(q["query"]))
            print(" plan", json.dumps(plan))
            print(" rows", [len(c[0]) for c in cols])
            if bad >= 3:
                sys.exit(0)
        qq.close()
        for r in rels:
            r.close()
print("done, bad =", bad)
