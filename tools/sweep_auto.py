#!/usr/bin/env python
"""Time every greedy schedule (K1 stream, K1b bucket, K1g grid) over a grid of
(batch, n) shapes with iters = n/4 to place AUTO's switch points.  One JSON
line per shape: {"B", "n", "iters", "<sched>_ms"...}.  CUDA events, median of 3."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device  # noqa: E402


def timed(x, n, iters, reps=3, out_dtype=None):
    B = x.shape[0]
    order = torch.empty((B, iters), dtype=torch.int64, device=x.device)
    sel = torch.empty((B, iters), dtype=out_dtype or x.dtype, device=x.device)
    seeds = torch.zeros(B, dtype=torch.int64, device=x.device)
    _device.greedy(x, n, iters, seeds, order, sel)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _device.greedy(x, n, iters, seeds, order, sel)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts)), order.cpu()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, nargs="*", default=[1, 4, 8, 16, 32, 64, 128])
    ap.add_argument("--ns", type=int, nargs="*", default=[4096, 8192, 16384, 32768, 65536, 131072])
    ap.add_argument("--scheds", nargs="*", default=["stream", "bucket", "grid", "auto"])
    ap.add_argument("--precision", choices=["f32", "f64"], default="f32",
                    help="f64: binary64 on the float coordinates (FFPS_F32_F64)")
    ap.add_argument("--iters-div", type=int, default=4, help="iterations = n / this")
    a = ap.parse_args()
    od = torch.float64 if a.precision == "f64" else None
    g = torch.Generator(device="cuda").manual_seed(0)
    for B in a.batches:
        for n in a.ns:
            x = torch.rand((B, n, 3), generator=g, device="cuda", dtype=torch.float64).float()
            iters = max(2, n // a.iters_div)
            row = {"B": B, "n": n, "iters": iters, "precision": a.precision}
            ref = None
            for s in a.scheds:
                if s == "auto":
                    os.environ.pop("FFPS_ALGO", None)
                    os.environ.pop("FFPS_GRID_CL", None)
                else:
                    os.environ["FFPS_ALGO"] = s.split("@")[0]
                    if "@" in s:
                        os.environ["FFPS_GRID_CL"] = s.split("@")[1]
                    else:
                        os.environ.pop("FFPS_GRID_CL", None)
                try:
                    ms, o = timed(x, n, iters, out_dtype=od)
                except Exception as ex:  # noqa: BLE001
                    row[s + "_ms"] = str(ex)[:60]
                    continue
                row[s + "_ms"] = round(ms, 3)
                if ref is None:
                    ref = o
                elif not torch.equal(ref, o):
                    row[s + "_mismatch"] = True
            os.environ.pop("FFPS_ALGO", None)
            os.environ.pop("FFPS_GRID_CL", None)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
