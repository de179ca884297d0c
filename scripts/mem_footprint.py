"""Device memory held by one query of a config (relations + trie storage +
frontier buffers after one execution): python scripts/mem_footprint.py [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_10841_b200 as fjg
from paper_2301_10841_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "scale_triangle"
torch.cuda.init()
eng = fjg.Engine(0)
free0, total = torch.cuda.mem_get_info()
w = configs.CONFIGS[name]()
q, _, rels = fjg.prepare_workload(eng, w)
eng.sync()
free1, _ = torch.cuda.mem_get_info()
r = q.execute(output_mode=w.output_mode)
eng.sync()
free2, _ = torch.cuda.mem_get_info()
GB = 1 << 30
print(f"{name}: relations + trie storage {(free0 - free1) / GB:.1f} GiB, after one execution {(free0 - free2) / GB:.1f} GiB "
      f"of {total / GB:.0f} GiB; count {r.count}")
