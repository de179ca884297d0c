"""Sharded-path step breakdown at one rank (fjg_execute_multi over NCCL, world
1): exchange / reduce device time per step, then the warm-step CUPTI kernel
timeline.
Usage: python scripts/shard_timeline.py [config]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs, dist as D
from paper_2301_10841_b200 import plan as P

name = sys.argv[1] if len(sys.argv) > 1 else "triangle"
torch.cuda.set_device(0)
eng = fjg.Engine(0)
w = configs.CONFIGS[name]()
plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
comm = D.Comm(eng, 1, 0)
sq = D.ShardedQuery(eng, w, plan, comm)
for _ in range(5):
    sq.execute(output_mode=w.output_mode)
for _ in range(3):
    t0 = time.perf_counter()
    r = sq.execute(output_mode=w.output_mode, timing=True)
    t1 = time.perf_counter()
    print(f"step {1e3*(t1-t0):.3f} ms (host wall)  exchange {r.extra['exchange_ms']:.3f} ms  "
          f"reduce {r.extra['reduce_ms']:.3f} ms  build {r.build_ms:.3f}  join {r.join_ms:.3f}  syncs {r.host_syncs}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sq.execute(output_mode=w.output_mode)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
for e in evs[:60]:
    gap = e.time_range.start - prev_end
    print(f"{(e.time_range.start - t0):9.1f} us  +gap {gap:7.1f}  dur {e.time_range.elapsed_us():8.1f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
sq.close()
comm.close()
