"""Device time of one execution in count vs enumerate mode (single pass: the
enumerate pass folds count / checksum too), CUDA events on the engine stream.
python scripts/enum_vs_count.py [config]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "chain"
eng = fjg.Engine(0)
stream = torch.cuda.ExternalStream(eng.stream_ptr, device=torch.device("cuda", 0))
w = configs.CONFIGS[name]()
q, _, _ = fjg.prepare_workload(eng, w)


def timed(mode, n=20):
    for _ in range(3):
        r = q.execute(output_mode=mode)
    ms = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = q.execute(output_mode=mode)
        e1.record(stream)
        eng.sync()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms), r


c_ms, c = timed("count")
e_ms, e = timed("enumerate")
print(f"{name}: count {c_ms:.3f} ms, enumerate {e_ms:.3f} ms ({e_ms / c_ms:.2f}x), rows {e.output_rows} == count {c.count}:"
      f" {e.output_rows == c.count}, checksum equal: {e.checksum == c.checksum}")
