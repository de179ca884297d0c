"""bench.py harness on the CPU: the --gpus N launcher (re-exec under
torch.distributed.run, world size N, rank 0 prints one line) and the
oracle-only reference arm (no product library loaded, same config dict as the
GPU arm, result printed)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return lines


def test_launcher_world2_reference():
    lines = _run(["--gpus", "2", "--impl", "reference", "--config", "chain", "--small", "--steps", "1",
                  "--warmup", "0", "--cpu-threads", "2"])
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["impl"] == "reference"


@pytest.mark.parametrize("cfg", ["chain", "triangle", "star", "path5"])
def test_reference_arm_oracle_only(cfg):
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', %r, '--small', "
            "'--steps', '1', '--warmup', '0', '--cpu-threads', '2']; runpy.run_path('bench.py', run_name='__main__');"
            "import os; root = os.path.realpath('.'); maps = open('/proc/self/maps').read(); "
            "print('LOADED', sorted({os.path.relpath(l.split()[-1], root) for l in maps.splitlines() "
            "if l.split()[-1].startswith(root) and l.split()[-1].endswith('.so')}))") % cfg
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    loaded = [x for x in r.stdout.splitlines() if x.startswith("LOADED")][0]
    assert "libfjg.so" not in loaded and "libfjgen.so" not in loaded, loaded
    assert "oracle/liboracle.so" in loaded and "paper_2301" not in loaded, loaded
    from paper_2301_10841_b200 import configs
    sys.path.insert(0, ROOT)
    import bench
    w = bench.workload(cfg, small=True)
    assert line["config"] == bench.config_dict(w.name, w.params, w.mode, "colt")
    assert line["result"]["scope"] == "whole query"
    from oracle import oracle
    from paper_2301_10841_b200 import plan as P
    plan = P.compile_plan({"query": w.query, "binary_plan": w.binary_plan}, w.mode)
    mv = P.head_variables(w.query).index(w.min_var) if w.min_var else -1
    ref = oracle.execute(w.query, plan, w.atom_columns(), output_mode=w.output_mode, min_var=mv)
    assert line["result"]["count"] == ref["count"] and line["result"]["checksum"] == f"{ref['checksum']:#018x}"
    assert configs  # product configs imported only here, in the checking process
