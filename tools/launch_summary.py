"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count and total."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path):
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("mr::<unnamed>::", "")
        ms = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:6d} {t:10.3f} ms {100 * t / tot:5.1f}%  {n}")
    print(f"total {tot:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
