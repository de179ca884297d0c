"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        if d.get("Metric Unit") == "ms":
            v *= 1e6
        elif d.get("Metric Unit") == "us":
            v *= 1e3
        k = d["Kernel Name"].split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1] / 1e6:10.3f} ms {100 * v[1] / tot:5.1f}% n={v[0]:4d} {k}")


if __name__ == "__main__":
    main(sys.argv[1])
