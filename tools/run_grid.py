#!/usr/bin/env python
"""One greedy launch of the C5 FlashFPS stage (B=64, n=50,000, k=12,500) under
a chosen schedule — a minimal target for ncu captures."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--n", type=int, default=50000)
ap.add_argument("--iters", type=int, default=12500)
ap.add_argument("--sched", default="grid@2")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((a.batch, a.n, 3), generator=g, device="cuda", dtype=torch.float64).float()
_device.set_schedule(a.sched)
order = torch.empty((a.batch, a.iters), dtype=torch.int64, device="cuda")
sel = torch.empty((a.batch, a.iters), dtype=x.dtype, device="cuda")
seeds = torch.zeros(a.batch, dtype=torch.int64, device="cuda")
for _ in range(a.reps):
    _device.greedy(x, a.n, a.iters, seeds, order, sel)
torch.cuda.synchronize()
print("ok", int(order[0, -1]))
