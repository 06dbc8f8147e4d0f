"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel.
Usage: python tools/launches.py launches.csv [--last-fraction 0.5]"""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
    return [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]]


def short(name):
    name = name.replace("void ", "")
    base = name.split("(")[0]
    return base[:60]


def summary(data):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, k, v in data:
        agg[short(k)][0] += 1
        agg[short(k)][1] += v
    tot = sum(v[1] for v in agg.values())
    return agg, tot


if __name__ == "__main__":
    data = load(sys.argv[1])
    frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    data = data[int(len(data) * (1 - frac)):]
    agg, tot = summary(data)
    print(f"{'kernel':62s} {'n':>5s} {'ms':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:62s} {v[0]:5d} {v[1] / 1e6:9.3f} {100 * v[1] / tot:5.1f}%")
    print(f"total {tot / 1e6:.3f} ms over {len(data)} launches")
