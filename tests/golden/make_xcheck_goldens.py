"""Independent cross-checks and full-size goldens for the graph configs
(VERDICT r1 "next" #1, #9). Test infrastructure.

oracle/xcheck.cpp counts triangles / oriented 4-cliques / walks on a plain CSR
adjacency, independently of the Free Join oracle. This script
  1. checks xcheck against the oracle's committed full-size goldens for C2
     (triangle) and C4 (4-clique), and against the oracle's C5 partition golden
     (tests/golden/scale_partition.json: partition 0 of 256, E2 whole);
  2. computes the full C5 triangle result (R-MAT 2^27, 512M edges) and writes
     it into configs_full.json["scale_triangle"] (the oracle pins it only
     through (1): it was run on partition 0 of 256; xcheck agrees with it there
     and on the whole of C2 and C4);
  3. computes the C5 5-path walk count 1^T A^5 1 exactly: residues mod 2^64 and
     mod two ~2^61 primes, combined by CRT (modulus > 2^186 > the count),
     into configs_full.json["scale_path5"].
Runs on the CPU (host R-MAT generator, ~20 GB RAM); minutes on 8 cores.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle import xcheck  # noqa: E402
from paper_2301_10841_b200 import configs, plan as P  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs_full.json")
PART = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scale_partition.json")
PRIMES = (2305843009213693951, 2305843009213693921)  # 2^61 - 1 and 2^61 - 31 (both prime)


def crt(residues, moduli):
    x, m = 0, 1
    for r, p in zip(residues, moduli):
        t = ((r - x) * pow(m, -1, p)) % p
        x, m = x + m * t, m * p
    return x, m


def main():
    gold = json.load(open(GOLD))
    t0 = time.time()
    for name, fn in (("triangle", xcheck.triangles), ("clique4", xcheck.clique4)):
        w = configs.CONFIGS[name]()
        r = fn(*w.relations["E"])
        assert r["count"] == gold[name]["count"] and f"{r['checksum']:#018x}" == gold[name]["checksum"], (name, r)
        print(name, "xcheck == oracle golden", r["count"], f"{time.time() - t0:.1f}s", flush=True)
    w = configs.scale_triangle()
    src, dst = w.relations["E"]
    print("C5 generated", len(src), f"{time.time() - t0:.1f}s", flush=True)
    pg = json.load(open(PART))
    r = xcheck.triangles(src, dst, nparts=pg["G"], part=pg["r"])
    assert r["count"] == pg["count"] and f"{r['checksum']:#018x}" == pg["checksum"], r
    print("C5 partition", pg["r"], "of", pg["G"], "xcheck == oracle", r["count"], f"{time.time() - t0:.1f}s", flush=True)
    t1 = time.time()
    r = xcheck.triangles(src, dst)
    tri_s = time.time() - t1
    print("C5 triangle", r, f"{tri_s:.1f}s", flush=True)
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    gold["scale_triangle"] = {
        "params": w.params, "count": r["count"], "checksum": f"{r['checksum']:#018x}", "min": None,
        "input_tuples": w.input_tuples(), "plan": plan, "source": "xcheck (oracle/xcheck.cpp, CSR bitmap counter)",
        "pinned_by": "xcheck == oracle on C2, C4 (whole) and on C5 partition 0 of 256 (scale_partition.json)",
        "xcheck_seconds": round(tri_s, 1), "xcheck_threads": os.cpu_count()}
    t1 = time.time()
    res = xcheck.walks(src, dst, 5, PRIMES)
    exact, modulus = crt(res, (2 ** 64,) + PRIMES)
    print("C5 5-path walks", exact, f"{time.time() - t1:.1f}s", flush=True)
    assert exact < modulus // 2
    wp = configs.scale_path5()
    gold["scale_path5"] = {
        "params": wp.params, "count": exact, "residues": {"2^64": res[0], str(PRIMES[0]): res[1], str(PRIMES[1]): res[2]},
        "input_tuples": wp.input_tuples(), "source": "xcheck walks 1^T A^5 1 (CSR SpMV), exact by CRT"}
    with open(GOLD, "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print("written", GOLD)


if __name__ == "__main__":
    main()
