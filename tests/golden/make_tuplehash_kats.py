"""Generate tests/golden/tuplehash_kats.json by running the reference's own
TupleHash (proj/include/fj/value.hpp:61-67) compiled as-is from
/root/reference (oracle/_ref/ref_kat, built by oracle/build_ref.sh).
Test infrastructure; run in the build container where /root/reference exists.
"""
import json
import os
import random
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
KAT = os.path.join(ROOT, "oracle", "_ref", "ref_kat")


def cases():
    fixed = [[], [0], [1, 2, 3], [1, 2, 3, 4], [-1, 0], [1048575, 1048575], [2, 1, 3],
             [2147483647, -2147483648], [-2147483648], [0, 0, 0, 0, 0, 0]]
    rng = random.Random(2301_10841)
    rnd = []
    for _ in range(60):
        n = rng.randint(0, 6)
        rnd.append([rng.randint(-2 ** 31, 2 ** 31 - 1) for _ in range(n)])
    for _ in range(10):  # int64 Values beyond int32 (oracle side only)
        n = rng.randint(1, 4)
        rnd.append([rng.randint(-2 ** 63, 2 ** 63 - 1) for _ in range(n)])
    return fixed + rnd


def main():
    if not os.path.exists(KAT):
        subprocess.check_call(["sh", os.path.join(ROOT, "oracle", "build_ref.sh")])
    cs = cases()
    inp = "".join(f"{len(t)} " + " ".join(map(str, t)) + "\n" for t in cs)
    out = subprocess.run([KAT], input=inp, capture_output=True, text=True, check=True).stdout.split()
    kats = [{"tuple": t, "hash": h} for t, h in zip(cs, out)]
    with open(os.path.join(HERE, "tuplehash_kats.json"), "w") as f:
        json.dump({"source": "fj::TupleHash from /root/reference/proj/include/fj/value.hpp (g++ 13, libstdc++)",
                   "kats": kats}, f, indent=1)
    print(len(kats), "KATs")


if __name__ == "__main__":
    main()
