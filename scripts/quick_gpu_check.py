"""Quick parity sweep: small configs + random plans on the GPU vs the CPU oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs
from oracle import oracle

eng = fjg.Engine(0)
cases = [configs.chain(n=20000, domain=20000), configs.triangle(scale=12, m=30000, seed=3),
         configs.star(nf=200000, dims=(20000, 30000, 8000, 1000)), configs.clique4(scale=12, m=40000)]
for w in cases:
    t0 = time.time()
    res, q, plan, _ = fjg.run_workload(eng, w)
    t1 = time.time()
    ref = oracle.execute(w.query, plan, w.atom_columns(), min_var=(q.head.index(w.min_var) if w.min_var else -1))
    ok = res.count == ref["count"] and res.checksum == ref["checksum"] and res.min_value == ref["min"]
    print(w.name, "OK" if ok else "MISMATCH", res.count, ref["count"], hex(res.checksum), hex(ref["checksum"]),
          res.min_value, ref["min"], f"gpu {t1-t0:.3f}s launches={res.kernel_launches} syncs={res.host_syncs}",
          flush=True)
