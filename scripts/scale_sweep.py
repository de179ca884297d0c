"""Last-node throughput vs table size: R-MAT triangles at several scales
(probed level-1 table = 32 B x edges; L2 = 126 MB). Prints candidates/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs

eng = fjg.Engine(0)
for scale, m in [(18, 1 << 20), (19, 1 << 21), (20, 1 << 22), (21, 1 << 23), (22, 1 << 24)]:
    w = configs.triangle(scale=scale, m=m)
    q, _, _ = fjg.prepare_workload(eng, w)
    for _ in range(3):
        r = q.execute(timing=True)
    ts = []
    for _ in range(5):
        r = q.execute(timing=True)
        ts.append(r.last_node_ms)
    t = sorted(ts)[2]
    print(f"scale {scale} edges {m}: table {32*m/2**20:.0f} MB  candidates {r.last_node_candidates:.3e}  "
          f"last {t:.3f} ms  {r.last_node_candidates/t/1e6:.3f} Gcand/s  step-ish build {r.build_ms:.3f}", flush=True)
    q.close()
