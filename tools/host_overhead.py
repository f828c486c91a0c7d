#!/usr/bin/env python
"""Host (CPU) time to enqueue one C5 FlashFPS step through the host pipeline
and through the device API, with the GPU busy: what the Python + C-ABI layers
add before the last chunk's kernels can start."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402
from paper_2604_17720_b200 import batched  # noqa: E402

B, N, budgets = 64, 200000, (50000, 12500, 3125, 781)
host = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).pin_memory()
x = host.cuda()
cfg = ffps.PruneConfig(p=0.75)
oi = torch.empty((B, budgets[0]), dtype=torch.int64).pin_memory()
os_ = torch.empty((B, budgets[0]), dtype=torch.float64).pin_memory()
for _ in range(3):
    ffps.hierarchical_sample_host(host, budgets, cfg, out=(oi, os_), precision="f64")

# device API: CPU time of the enqueue (the kernels run asynchronously)
ts = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ffps.hierarchical_sample_batch(x, budgets, cfg, 0, True, precision="f64")
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print(f"device API enqueue: median {np.median(ts) * 1e3:.3f} ms")

# host pipeline: patch the final synchronize to time the enqueue part
orig = torch.cuda.Stream.synchronize
marks = []


def timed_sync(self):
    marks.append(time.perf_counter())
    return orig(self)


torch.cuda.Stream.synchronize = timed_sync
ts = []
for _ in range(10):
    torch.cuda.synchronize()
    marks.clear()
    t0 = time.perf_counter()
    ffps.hierarchical_sample_host(host, budgets, cfg, out=(oi, os_), precision="f64")
    t1 = time.perf_counter()
    ts.append(((marks[-1] if marks else t1) - t0, t1 - t0))
torch.cuda.Stream.synchronize = orig
print(f"host pipeline: enqueue {np.median([a for a, _ in ts]) * 1e3:.3f} ms, "
      f"wall {np.median([b for _, b in ts]) * 1e3:.3f} ms")
