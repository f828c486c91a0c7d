#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total / mean device time and share of the total."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3}.get(r[iu], 1.0)
        name = r[ik]
        agg[name.split("(")[0][:90]].append(v)   # msecond
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':92s} {'n':>5s} {'total_ms':>10s} {'mean_ms':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:92s} {len(v):5d} {sum(v):10.3f} {sum(v)/len(v):10.4f} {sum(v)/tot:6.1%}")
    print(f"total device time {tot:.3f} ms over {sum(len(v) for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
