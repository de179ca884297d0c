"""Sharded-path step breakdown at one rank (NCCL, world 1): host wall time of
exchange / query / reduce per step, then the warm-step CUPTI kernel timeline.
Usage: python scripts/shard_timeline.py [config]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
import torch
import torch.distributed as dist
from torch.profiler import profile, ProfilerActivity
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs, dist as D
from paper_2301_10841_b200 import plan as P

name = sys.argv[1] if len(sys.argv) > 1 else "triangle"
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
eng = fjg.Engine(0)
w = configs.CONFIGS[name]()
plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
sq = D.ShardedQuery(eng, w, plan, 1, 0)
for _ in range(5):
    sq.execute(output_mode=w.output_mode)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    held = D.exchange(sq.local, sq.views, 1, 0, sq.ops, None, sq._held)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = sq._q.execute(output_mode=w.output_mode)
    t2 = time.perf_counter()
    D.reduce_results(r.count, r.checksum, r.min_value, sq.ops.device)
    t3 = time.perf_counter()
    print(f"exchange {1e3*(t1-t0):.3f} ms  query {1e3*(t2-t1):.3f} ms  reduce {1e3*(t3-t2):.3f} ms")
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
dist.destroy_process_group()
