"""Warm-step kernel timeline of one C2 execute via torch.profiler (CUPTI):
per-kernel device time and the idle gaps between kernels (host syncs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "triangle"
eng = fjg.Engine(0)
w = configs.CONFIGS[name]()
q, _, _ = fjg.prepare_workload(eng, w)
for _ in range(5):
    q.execute(output_mode=w.output_mode)
eng.sync()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    q.execute(output_mode=w.output_mode)
    eng.sync()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
tot_gap = 0.0
for e in evs:
    gap = e.time_range.start - prev_end
    tot_gap += max(gap, 0)
    print(f"{(e.time_range.start - t0):9.1f} us  +gap {gap:7.1f}  dur {e.time_range.elapsed_us():8.1f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
print(f"span {prev_end - t0:.1f} us, gaps {tot_gap:.1f} us, kernels+copies {sum(e.time_range.elapsed_us() for e in evs):.1f} us")
agg = {}
for e in evs:
    k = e.name[:60]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += e.time_range.elapsed_us()
print("---- per kernel ----")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t:10.1f} us  n={n:4d}  {k}")
