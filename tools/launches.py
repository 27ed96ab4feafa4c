"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per-kernel totals)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
        v = float(d["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += v
    return agg


if __name__ == "__main__":
    agg = load(sys.argv[1])
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':48s} {'n':>5s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} {c:5d} {v:10.1f} {v / c:9.2f} {100 * v / tot:5.1f}%")
    print(f"{'TOTAL':48s} {sum(c for c, _ in agg.values()):5d} {tot:10.1f}")
