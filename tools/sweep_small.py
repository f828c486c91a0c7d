#!/usr/bin/env python
"""K1s configurations (threads, points per thread) per cloud size: ns per greedy
step, CUDA events, median of 5 (FFPS_SMALL_PLAN forces one)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device  # noqa: E402
from tools.sweep_auto import timed  # noqa: E402

PLANS = ["256,8", "256,16", "256,24", "256,32"]  # the compiled float configurations
_device.set_schedule("small")
for B, n in [(16, 2048), (1, 4096), (64, 3125), (16, 6000), (64, 8000)]:
    it = n // 4
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((B, n, 3), generator=g, device="cuda", dtype=torch.float64).float()
    ref = None
    for pl in PLANS:
        nt, q = map(int, pl.split(","))
        if nt * q < n:
            continue
        os.environ["FFPS_SMALL_PLAN"] = pl
        ms, order = timed(x, n, it, reps=5)
        same = ref is None or bool(torch.equal(order, ref))
        ref = order if ref is None else ref
        print(f"B={B} n={n} plan={pl:8s} {ms * 1e6 / it:5.0f} ns/step same={same}", flush=True)
    os.environ.pop("FFPS_SMALL_PLAN", None)
