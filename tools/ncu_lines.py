#!/usr/bin/env python
"""Aggregate warp-stall samples of an ncu report per CUDA source line
(ncu -i X --page source --csv --print-source cuda,sass > X.csv) and print the
hottest lines with their top stall reasons."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    tot = defaultdict(int)
    rs = defaultdict(lambda: defaultdict(int))
    src = {}
    fname = "?"
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = {k: i for i, k in enumerate(r)}
            reasons = [(i, k) for i, k in enumerate(r) if k.startswith("stall_") and "Not Issued" not in k]
            continue
        if hdr is None or not r[0].isdigit():
            continue
        key = (fname, int(r[0]))
        src[key] = r[1]
        try:
            smp = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, IndexError):
            continue
        tot[key] += smp
        for i, k in reasons:
            try:
                rs[key][k[6:]] += int(r[i] or 0)
            except ValueError:
                pass
    all_s = sum(tot.values())
    print("total samples", all_s)
    for key, v in sorted(tot.items(), key=lambda t: -t[1])[:top]:
        top3 = sorted(rs[key].items(), key=lambda t: -t[1])[:3]
        print(f"{key[0]}:{key[1]:<5d} {v:7d} {100.0 * v / all_s:5.1f}%  {src[key].strip()[:70]:70s} "
              + " ".join(f"{k}={n}" for k, n in top3 if n))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
