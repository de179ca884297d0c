"""Generate tests/golden/configs_full.json: the CPU oracle's count / checksum /
MIN for every BASELINE.json config at full size (seeded inputs from
paper_2301_10841_b200/configs.py). Test infrastructure: the GPU parity tests
compare the device results against these committed numbers, so the GPU box
never has to rerun the oracle at full size.

    python tests/golden/make_config_goldens.py [config ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2301_10841_b200 import configs, plan as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs_full.json")


def main(names):
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        w = configs.CONFIGS[name]()
        plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
        head = P.head_variables(w.query)
        mv = head.index(w.min_var) if w.min_var else -1
        t0 = time.time()
        nt = int(os.environ.get("GOLDEN_THREADS", os.cpu_count() or 1))
        r = oracle.execute(w.query, plan, w.atom_columns(), min_var=mv, nthreads=nt)
        dt = time.time() - t0
        res[name] = {"params": w.params, "plan": plan, "count": r["count"], "checksum": f"{r['checksum']:#018x}",
                     "min": r["min"], "probes": r["probes"], "input_tuples": w.input_tuples(),
                     "oracle_seconds": round(dt, 1), "oracle_threads": nt}
        print(name, res[name]["count"], res[name]["checksum"], f"{dt:.1f}s", flush=True)
        with open(OUT, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["chain", "triangle", "star", "clique4"])
