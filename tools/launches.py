"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total and mean duration (cold-cache, serialised
launches: use the shares, not the absolutes)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
         "ms": 1e3, "msecond": 1e3}


def summarise(path):
    hdr = None
    agg = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        us = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    tot = sum(t for _, t in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:58]:58s} {n:4d} {t/1e3:9.2f} ms  mean {t/n:9.1f} us  {100*t/tot:5.1f}%")
