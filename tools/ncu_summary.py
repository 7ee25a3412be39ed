"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) per kernel: python tools/ncu_summary.py file.csv"""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "")
            v = float(r[vi].replace(",", ""))
            v = v / 1000.0 if r[ui] == "ns" else (v * 1000.0 if r[ui] == "ms" else v)   # -> us
            agg.setdefault(name, []).append(v)
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    print(f"{'kernel':36s} {'n':>5s} {'mean_us':>10s} {'min_us':>10s} {'max_us':>10s}")
    for k, v in agg.items():
        print(f"{k:36s} {len(v):5d} {sum(v)/len(v):10.2f} {min(v):10.2f} {max(v):10.2f}")
