import torch, time
for mb in (16, 64, 256):
    n = mb * 2**20 // 4
    h = torch.empty(n, dtype=torch.int32).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(mb, "MB", 5 * mb / 1024 / (e0.elapsed_time(e1) / 1000), "GB/s")
# two streams
n = 16 * 2**20 // 4
hs = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(2)]
ds = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(2)]
ss = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    for h, d, s in zip(hs, ds, ss):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print("2 streams x 16MB x5", 5 * 32 / 1024 / dt, "GB/s")
# engine relation create from pinned host columns (alloc + copy)
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_10841_b200 as fjg
eng = fjg.Engine(0)
st = torch.cuda.ExternalStream(eng.stream_ptr)
n = 4194304
hc = [torch.randint(0, 1 << 20, (n,), dtype=torch.int32).pin_memory() for _ in range(2)]
for it in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.sync(); e0.record(st)
    r = eng.relation_host_ptrs([c.data_ptr() for c in hc], n)
    e1.record(st); eng.sync()
    print("relation_create 2x16MB", e0.elapsed_time(e1), "ms")
    r.close()
