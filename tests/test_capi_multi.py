"""fjg_execute_multi from a compiled C++ caller (tests/capi_multi_main.cpp,
g++ against include/fjg.h and libfjg.so; no Python in the process that runs
the query) at world size 1 on the GPU, against the oracle. The CPU test only
compiles and links it."""
import json
import os
import struct
import subprocess

import numpy as np
import pytest

from oracle import oracle
from paper_2301_10841_b200 import _capi, configs, dist as D, plan as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_caller(out_dir):
    exe = os.path.join(out_dir, "capi_multi_main")
    lib = os.path.abspath(_capi.LIB_PATH)  # the library this process loaded (FJG_LIB honoured)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "capi_multi_main.cpp"), lib,
                    f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", exe], check=True)
    return exe


def write_workload(path, w, plan):
    bases = sorted(set(w.atom_rel))
    rels = w.filtered()
    _, views = D.atom_views(w.query, w.atom_rel, plan)
    head = P.head_variables(w.query)
    with open(path, "wb") as f:
        f.write(struct.pack("<i", len(bases)))
        for b in bases:
            cols = rels[b]
            f.write(struct.pack("<iQ", len(cols), len(cols[0])))
            for c in cols:
                f.write(np.ascontiguousarray(c, dtype=np.int32).tobytes())
        f.write(struct.pack("<i", len(w.atom_rel)))
        f.write(struct.pack(f"<{len(w.atom_rel)}i", *[bases.index(b) for b in w.atom_rel]))
        f.write(struct.pack(f"<{len(w.atom_rel)}i", *[-1 if c is None else c for (_, c) in views]))
        f.write(struct.pack("<ii", {"count": 0, "factorized_count": 2}[w.output_mode],
                            head.index(w.min_var) if w.min_var else -1))
        for s in (json.dumps({"query": w.query}), json.dumps([[[r, list(v)] for (r, v) in n] for n in plan])):
            b = s.encode()
            f.write(struct.pack("<Q", len(b)) + b)


def test_caller_compiles(tmp_path):
    assert os.access(build_caller(str(tmp_path)), os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["triangle", "star", "chain", "clique4", "path5"])
def test_compiled_caller_world1(tmp_path, name):
    w = {"triangle": lambda: configs.triangle(scale=12, m=30000, seed=3),
         "star": lambda: configs.star(nf=200000, dims=(3000, 4000, 800, 100)),
         "chain": lambda: configs.chain(n=20000, domain=30000),
         "clique4": lambda: configs.clique4(scale=11, m=20000),
         "path5": lambda: configs.path5(scale=11, m=12000)}[name]()
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    exe = build_caller(str(tmp_path))
    data = os.path.join(str(tmp_path), "w.bin")
    write_workload(data, w, plan)
    p = subprocess.run([exe, data], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr + p.stdout
    head = P.head_variables(w.query)
    ref = oracle.execute(w.query, plan, w.atom_columns(), min_var=head.index(w.min_var) if w.min_var else -1,
                         output_mode=w.output_mode)
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 2
    for r in lines:
        assert (r["count_hi"] << 64 | r["count_lo"]) == ref["count"]
        if w.output_mode == "count":
            assert r["checksum"] == ref["checksum"]
        assert (r["min"] if r["has_min"] else None) == ref["min"]
