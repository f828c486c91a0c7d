#!/usr/bin/env python
"""cProfile of the host side of hierarchical_sample_batch (C5, binary64): the
Python + ctypes work that precedes the first kernel of every step."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402

B, N, budgets = 64, 200000, (50000, 12500, 3125, 781)
x = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).cuda()
cfg = ffps.PruneConfig(p=0.75)
for _ in range(3):
    ffps.hierarchical_sample_batch(x, budgets, cfg, 0, True, precision="f64")
torch.cuda.synchronize()
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ffps.hierarchical_sample_batch(x, budgets, cfg, 0, True, precision="f64")
    ts.append(time.perf_counter() - t0)
print(f"enqueue per call (GPU idle at entry): median {np.median(ts) * 1e6:.1f} us")
pr = cProfile.Profile()
for _ in range(30):
    torch.cuda.synchronize()
    pr.enable()
    ffps.hierarchical_sample_batch(x, budgets, cfg, 0, True, precision="f64")
    pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
