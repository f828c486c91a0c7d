#!/usr/bin/env python
"""Streaming kernel (K1) on small clouds: time forced plans (nt,p,s,C) against
the planner's choice for the C1 / C2-flash shapes.  CUDA events, median of 5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device  # noqa: E402
from tools.sweep_auto import timed  # noqa: E402

SHAPES = [(16, 6000, 1500), (1, 4096, 1024), (16, 3000, 750), (64, 3125, 781), (64, 8000, 2000),
          (128, 4096, 1024)]
PLANS = ["", "small", "256,4,0,6", "256,8,0,3", "256,16,8,1"]
for B, n, it in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((B, n, 3), generator=g, device="cuda", dtype=torch.float64).float()
    ref = None
    for pl in PLANS:
        _device.set_schedule("small" if pl == "small" else "stream")
        os.environ["FFPS_FORCE_PLAN"] = "" if pl == "small" else pl
        try:
            ms, order = timed(x, n, it, reps=5)
        except Exception as e:  # noqa: BLE001
            print(f"B={B} n={n} plan={pl or 'auto'}: {str(e)[:60]}")
            continue
        same = ref is None or bool(torch.equal(order, ref))
        ref = order if ref is None else ref
        print(f"B={B} n={n} plan={pl or 'auto':12s} {ms:.3f} ms  {ms * 1e6 / it:.0f} ns/iter  same={same}",
              flush=True)
    os.environ.pop("FFPS_FORCE_PLAN", None)
