"""Re-run one stress case (scripts/stress_parity.py's last-case JSON) against the oracle."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import plan as P
from oracle import oracle

d = json.load(open(sys.argv[1]))
q = d["q"]
cols = [[np.array(c, dtype=np.int32) for c in cs] for cs in d["cols"]]
plan = P.compile_plan(q, d["mode"])
print("plan", plan, flush=True)
mv = d["mv"]
ref = oracle.execute(q, plan, cols, min_var=mv, dynamic_cover=d["dyn"], backend=d["backend"])
eng = fjg.Engine(0)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    rels = [eng.relation(c) for c in cols]
    qq = eng.query({"query": q["query"]}, plan, rels)
    r = qq.execute(batch_size=d["batch"], dynamic_cover=d["dyn"], backend=d["backend"], min_var=None if mv < 0 else mv)
    print(rep, r.count, ref["count"], hex(r.checksum), hex(ref["checksum"]), "keys", r.keys_inserted,
          ref["keys_inserted"], flush=True)
    qq.close()
    for x in rels:
        x.close()
