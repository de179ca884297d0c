"""Where the e2e step goes (C2): H2D, query build on the host, execute."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs, plan as P

eng = fjg.Engine(0)
stream = torch.cuda.ExternalStream(eng.stream_ptr, device=torch.device("cuda", 0))
w = configs.triangle()
host = {n: [torch.from_numpy(c).pin_memory() for c in cols] for n, cols in w.relations.items()}
for it in range(6):
    eng.sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record(stream)
    rels = {n: eng.relation_host_ptrs([c.data_ptr() for c in cols], cols[0].numel()) for n, cols in host.items()}
    ev[1].record(stream)
    t1 = time.perf_counter()
    q, _, _ = fjg.prepare_workload(eng, w, device_relations=rels)
    t2 = time.perf_counter()
    ev[2].record(stream)
    r = q.execute()
    ev[3].record(stream)
    eng.sync()
    t3 = time.perf_counter()
    q.close()
    for x in rels.values():
        x.close()
    print(f"h2d {ev[0].elapsed_time(ev[1]):.3f} ms  prepare(host) {1000*(t2-t1):.3f} ms  "
          f"gap {ev[1].elapsed_time(ev[2]):.3f}  execute {ev[2].elapsed_time(ev[3]):.3f} ms  "
          f"total dev {ev[0].elapsed_time(ev[3]):.3f}  wall {1000*(t3-t0):.3f}", flush=True)
