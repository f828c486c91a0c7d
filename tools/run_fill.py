#!/usr/bin/env python
"""One seeded random fill (K2r) at the C5 shape — a minimal ncu target."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17720_b200 as ffps  # noqa: E402
from paper_2604_17720_b200 import _device  # noqa: E402

B, N, m1, k = 64, 200000, 50000, 12500
g = torch.Generator(device="cuda").manual_seed(0)
order = torch.empty((B, m1), dtype=torch.int64, device="cuda")
order[:, :k] = torch.stack([torch.randperm(50000, generator=g, device="cuda")[:k] for _ in range(B)])
sel = torch.zeros((B, m1), dtype=torch.float32, device="cuda")
_device.fill_random(order, sel, N, k, m1, 3)
torch.cuda.synchronize()
print("ok", int(order[0, -1]))
