"""Write oracle/workload_plans.json: the Free Join plan of every config as the
product's host plan compiler produces it (binary2fj / factor / fj_to_gj,
SPEC.md:204-240), so the oracle-only reference arm of bench.py needs no
product library. tests/test_oracle_workloads.py re-checks it. Test infrastructure."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2301_10841_b200 import configs, plan as P  # noqa: E402

SMALL = {"chain": dict(n=100), "triangle": dict(scale=8, m=500), "star": dict(nf=1000, dims=(50, 40, 30, 20)),
         "clique4": dict(scale=8, m=500), "path5": dict(scale=8, m=500)}


def plans():
    out = {}
    for name, kw in SMALL.items():
        w = configs.CONFIGS[name](**kw)
        out[name] = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    return out


if __name__ == "__main__":
    with open(os.path.join(ROOT, "oracle", "workload_plans.json"), "w") as f:
        ps = plans()
        f.write("{\n" + ",\n".join(f" {json.dumps(k)}: {json.dumps(v)}" for k, v in ps.items()) + "\n}\n")
