#!/usr/bin/env python
"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
and duration from an `ncu --set full` report into profiles/traffic.json, keyed
by kernel name; bench.py reports it as roofline.traffic."""
import csv
import io
import json
import subprocess
import sys


def main(rep, out="profiles/traffic.json", label=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))

        def val(k):
            v = float(d[k].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1e-3, "ms": 1e-3,
                     "us": 1e-6, "ns": 1e-9,
                     "usecond": 1e-6, "nsecond": 1e-9, "second": 1}
            return v * scale.get(u[k], 1)
        name = d["Kernel Name"].split("(")[0]
        res[name] = {"dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                     "duration_s": val("gpu__time_duration.sum"),
                     "grid": d.get("Grid Size"), "block": d.get("Block Size"),
                     "source": rep, "label": label}
    try:
        old = json.load(open(out))
    except (OSError, ValueError):
        old = {}
    old.update(res)
    json.dump(old, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
