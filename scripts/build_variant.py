"""Build libfjg.so variants with extra -D flags (perf experiments):
    python scripts/build_variant.py OUT.so -DFJG_GJ_R=4 ...
Run one with FJG_LIB=OUT.so python bench.py ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2301_10841_b200"))
import build as B  # noqa: E402

out, flags = sys.argv[1], sys.argv[2:]
B._run([B.NVCC, "-std=c++17", "-O3", *B.ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "128",
        *flags, *B._srcs("engine.cu", "capi.cpp", "fj_plan.cpp"), "-o", out])
print("built", out, *flags)
