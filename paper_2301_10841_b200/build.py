"""Build the native libraries in-tree (they travel to the GPU box with the repo).

  libfjg.so    product: host plan compiler + sm_100a executor + C-ABI (include/fjg.h)
  libfjgen.so  seeded synthetic data generators (bench / tests input)
  oracle/liboracle.so  CPU restatement (test infrastructure only)
  oracle/libxcheck.so  independent CSR graph counters (test infrastructure only)
  oracle/libogen.so    independent config input generators (reference arm / tests only)
  oracle/_ref/ref_kat  TupleHash KAT tool compiled from the reference header
                        (only when /root/reference is present)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

LIBFJG = os.path.join(HERE, "libfjg.so")
LIBFJGEN = os.path.join(HERE, "libfjgen.so")
LIBORACLE = os.path.join(ROOT, "oracle", "liboracle.so")
LIBXCHECK = os.path.join(ROOT, "oracle", "libxcheck.so")
LIBOGEN = os.path.join(ROOT, "oracle", "libogen.so")
REF_KAT = os.path.join(ROOT, "oracle", "_ref", "ref_kat")


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))


def _srcs(*names):
    return [os.path.join(CSRC, n) for n in names]


def build_product(force=False):
    kdir = os.path.join(CSRC, "kernels")
    deps = _srcs("engine.cu", "engine.cuh", "capi.cpp", "fj_plan.cpp", "fj_plan.hpp", "fj_json.hpp",
                 "fj_hash.hpp", "fj_errors.hpp", "multi.cuh", "colt_api.cuh") + [os.path.join(ROOT, "include", "fjg.h")] + \
        [os.path.join(kdir, f) for f in sorted(os.listdir(kdir)) if f.endswith(".cuh")]
    if force or _stale(LIBFJG, deps):
        _run([NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
              "-diag-suppress", "128",
              *_srcs("engine.cu", "capi.cpp", "fj_plan.cpp"), "-ldl", "-o", LIBFJG])
    gdeps = _srcs("datagen.cpp", "datagen_dev.cu", "rmat.hpp")
    if force or _stale(LIBFJGEN, gdeps):
        _run([NVCC, "-std=c++17", "-O3", *ARCH, "-Xcompiler", "-fPIC,-pthread,-march=x86-64-v2", "-shared",
              *_srcs("datagen.cpp", "datagen_dev.cu"), "-o", LIBFJGEN])


def build_oracle(force=False):
    src = os.path.join(ROOT, "oracle", "fj_oracle.cpp")
    if force or _stale(LIBORACLE, [src]):
        _run(["g++", "-std=c++17", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread", src,
              "-o", LIBORACLE])
    xsrc = os.path.join(ROOT, "oracle", "xcheck.cpp")
    if force or _stale(LIBXCHECK, [xsrc]):
        _run(["g++", "-std=c++17", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread", xsrc,
              "-o", LIBXCHECK])
    gsrc = os.path.join(ROOT, "oracle", "gen.cpp")
    if force or _stale(LIBOGEN, [gsrc]):
        _run(["g++", "-std=c++17", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread", gsrc,
              "-o", LIBOGEN])
    if os.path.isdir("/root/reference/proj/include"):
        kat = os.path.join(ROOT, "oracle", "ref_kat.cpp")
        if force or _stale(REF_KAT, [kat]):
            _run(["sh", os.path.join(ROOT, "oracle", "build_ref.sh")])


def build_all(force=False):
    build_product(force)
    build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built", LIBFJG, LIBFJGEN, LIBORACLE)
