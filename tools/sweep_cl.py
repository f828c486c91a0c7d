#!/usr/bin/env python
"""Greedy-stage time of the BASELINE FlashFPS / exhaustive stage-1 shapes
under the stream schedule and K1g with 1/2/4 CTAs per cloud (KM 16/8).
One JSON line per (shape, schedule).  CUDA events, median of 3."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device  # noqa: E402
from tools.sweep_auto import timed  # noqa: E402

SHAPES = [(16, 6000, 1500), (16, 24000, 6000), (8, 25000, 6250), (8, 100000, 25000),
          (32, 75000, 18750), (64, 50000, 12500)]
SCHEDS = ["stream", "grid@1", "grid@2", "grid@4", "grid@1/km8", "grid@2/km8"]
if len(sys.argv) > 1 and sys.argv[1] == "--grid":  # batch x n sweep, iters = n / 4
    SHAPES = [(b, n, n // 4) for b in (1, 2, 4, 8, 16, 32, 64, 128)
              for n in (8192, 12288, 16384, 24576, 50000, 100000, 200000)]
    SCHEDS = ["stream", "bucket", "grid@1", "grid@2", "grid@4"]

for B, n, it in SHAPES:
    if len(sys.argv) > 1 and sys.argv[1] != "--grid" and f"{B}x{n}" not in sys.argv[1:]:
        continue
    if B * n * it > 64 * 200000 * 50000:
        continue
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((B, n, 3), generator=g, device="cuda", dtype=torch.float64).float()
    ref = None
    for sc in SCHEDS:
        name, _, km = sc.partition("/km")
        os.environ.pop("FFPS_GRID_KM", None)
        if km:
            os.environ["FFPS_GRID_KM"] = km
        _device.set_schedule(name)
        try:
            ms, order = timed(x, n, it)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"B": B, "n": n, "iters": it, "sched": sc, "error": str(e)[:80]}))
            continue
        same = True if ref is None else bool(torch.equal(order, ref))
        ref = order if ref is None else ref
        print(json.dumps({"B": B, "n": n, "iters": it, "sched": sc, "ms": round(ms, 3),
                          "ns_per_iter": round(ms * 1e6 / it, 1), "same": same}), flush=True)
    os.environ.pop("FFPS_GRID_KM", None)
    _device.set_schedule("auto")
