#!/usr/bin/env python
"""One C5 FlashFPS stage-1 greedy call (64 clouds, 50,000-point candidate
prefix, 12,500 iterations; binary64 on float coordinates by default) after
one warm-up call: the short command the ncu captures of K0 + K1g profile."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17720_b200 as ffps  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
x = torch.from_numpy(np.stack([np.random.default_rng(b).random((50_000, 3)).astype(np.float32)
                               for b in range(64)])).cuda()
for _ in range(2):
    s, _ = ffps.fps_batch(x, 12_500, precision=None if prec == "f32" else "f64")
torch.cuda.synchronize()
print("ok", prec, int(s.indices[0, -1]))
