#!/usr/bin/env python
"""Per-kernel launch statistics (count, median, mean us) from an ncu
`--metrics gpu__time_duration.sum --csv` launch list.
python tools/launch_table.py LAUNCHES.csv"""
import collections
import csv
import sys


def table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    d = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        x = dict(zip(h, r))
        if x.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(x["Metric Value"].replace(",", ""))
        u = x.get("Metric Unit", "")
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        d[x["Kernel Name"]].append(v)
    out = []
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        vs = sorted(v)
        out.append((k, len(v), vs[len(vs) // 2], sum(v) / len(v)))
    return out


if __name__ == "__main__":
    for k, n, med, mean in table(sys.argv[1]):
        print(f"{k[:90]:90s} n={n:4d} median={med:9.2f} us mean={mean:9.2f} us")
