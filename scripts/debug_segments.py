import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import plan as P
from paper_2301_10841_b200.segments import run_segments, head_order
from paper_2301_10841_b200.configs import left_deep
from oracle import oracle
from randq import random_query, bag_equal
eng = fjg.Engine(0)
rng = np.random.default_rng(31)
tree = ["join", "A0", ["join", "A1", ["join", "A2", "A3"]]]
while True:
    q, cols = random_query(rng, max_atoms=4)
    if len(q["query"]) != 4: continue
    truth = oracle.brute_force(q, cols)
    if len(truth) > 20000: continue
    rels = {a["rel"]: eng.relation(c) for a, c in zip(q["query"], cols)}
    r, qq, trace = run_segments(eng, q["query"], tree, rels, mode="free", output_mode="enumerate")
    if not bag_equal(r.extra["rows"], truth):
        print("MISMATCH", q, [len(c[0]) for c in cols])
        for name, plan, rr in trace: print(name, plan, rr.count, rr.output_rows)
        # oracle per segment
        atoms = {a["rel"]: a for a in q["query"]}
        print("truth", len(truth))
        sub = oracle.brute_force({"query": [atoms["A2"], atoms["A3"]]}, [cols[2], cols[3]])
        print("P1 truth", len(sub))
        break
