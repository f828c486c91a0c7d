#!/usr/bin/env python
"""Print the SASS of an ncu report (page source --print-source sass, CSV) in
address order with stall samples and the top stall reasons, optionally only
lines whose execution count lies in [lo, hi] (e.g. warp-0-only code)."""
import csv
import sys


def main(path, lo=0, hi=1 << 62, top=0):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    out = []
    for r in rows[2:]:
        try:
            ex = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        if not lo <= ex <= hi:
            continue
        rs = sorted(((int(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
        out.append((r[ix["Address"]], r[ix["Source"]], smp, ex,
                    " ".join(f"{k}={v}" for v, k in rs if v)))
    if top:
        out.sort(key=lambda t: -t[2])
        out = out[:top]
    tot = sum(o[2] for o in out)
    for a, src, smp, ex, rs in out:
        print(f"{a:>6} {smp:6d} {ex:9d} {src[:60]:60s} {rs}")
    print("samples in selection:", tot)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], int(a[1]) if len(a) > 1 else 0, int(a[2]) if len(a) > 2 else 1 << 62,
         int(a[3]) if len(a) > 3 else 0)
