"""Generate tests/golden/scale_partition.json: the oracle's result for one
first-variable hash partition of the full-size C5 triangle (R-MAT 2^27,
512M edges): E1(a,b), E3(a,c) restricted to rows with partition_of(a, G) == r,
E2(b,c) the whole relation. The device runs the same restricted query in
tests/test_gpu_parity.py::test_scale_triangle_partition. Needs a GPU (the
2^27 graph is generated on the device, bit-identical to the host generator)
and ~60 GB host RAM. Test infrastructure.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2301_10841_b200 import configs, plan as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scale_partition.json")
G, R = 256, 0


def np_partition_of(v, nparts):
    with np.errstate(over="ignore"):
        k = v.astype(np.int64).astype(np.uint64) ^ np.uint64(0x5bd1e995)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xff51afd7ed558ccd)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xc4ceb9fe1a85ec53)
        k ^= k >> np.uint64(33)
    return (k % np.uint64(nparts)).astype(np.int64)


def restricted(w):
    src, dst = w.relations["E"]
    keep = np_partition_of(src, G) == R
    part = [src[keep], dst[keep]]
    return [part, [src, dst], part]


def main():
    t0 = time.time()
    w = configs.scale_triangle()
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    cols = restricted(w)
    print("generated", time.time() - t0, len(cols[0][0]), flush=True)
    t0 = time.time()
    r = oracle.execute(w.query, plan, cols)
    res = {"params": w.params, "G": G, "r": R, "rows_partition": int(len(cols[0][0])), "count": r["count"],
           "checksum": f"{r['checksum']:#018x}", "probes": r["probes"], "oracle_seconds": round(time.time() - t0, 1)}
    print(res, flush=True)
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
