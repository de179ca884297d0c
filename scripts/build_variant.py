"""Build a variant of libfjg.so with extra -D flags into variants/ (git-ignored)
for A/B timing on the GPU box:
    python scripts/build_variant.py variants/r4.so -DFJG_GJ_R=4 -DFJG_GJ_QC=256
then  bash scripts/run_variants.sh scale_triangle 3 default variants/r4.so"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2301_10841_b200"))
import build as B  # noqa: E402

out, flags = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
B._run([B.NVCC, "-std=c++17", "-O3", *B.ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "128",
        *flags, *B._srcs("engine.cu", "capi.cpp", "fj_plan.cpp"), "-ldl", "-o", out])
print("built", out, " ".join(flags))
