#!/usr/bin/env python
"""Where the C5 end-to-end time goes: the H2D copy of the candidate prefixes,
the device pipeline on resident clouds, the D2H of the results, the host-side
zeroing of the fill distances, and the chunked host pipeline (2/4/8 chunks)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402

B, N, budgets = 64, 200000, (50000, 12500, 3125, 781)
c, k = 50000, 12500
pinned = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).pin_memory()
cfg = ffps.PruneConfig(p=0.75)
oi = torch.empty((B, budgets[0]), dtype=torch.int64).pin_memory()
os_ = torch.empty((B, budgets[0]), dtype=torch.float64).pin_memory()
dev = torch.empty((B, c, 3), dtype=torch.float32, device="cuda")


def timed(fn, reps=7):
    ts = []
    for r in range(reps + 2):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(s.elapsed_time(e))
    return float(np.median(ts))


src = pinned[:, :c].contiguous().pin_memory()
print(f"H2D 38.4 MB (one contiguous pinned copy): {timed(lambda: dev.copy_(src, non_blocking=True)):.3f} ms")
xd = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).cuda()
print(f"device pipeline (resident clouds): "
      f"{timed(lambda: ffps.hierarchical_sample_batch(xd, budgets, cfg, 0, True, precision='f64')):.3f} ms")
gi = torch.zeros((B, budgets[0]), dtype=torch.int64, device="cuda")
gs = torch.zeros((B, k), dtype=torch.float64, device="cuda")
print(f"D2H 25.6 MB indices: {timed(lambda: oi.copy_(gi, non_blocking=True)):.3f} ms; "
      f"6.4 MB distances: {timed(lambda: os_[:, :k].copy_(gs, non_blocking=True)):.3f} ms")
t0 = time.perf_counter()
for _ in range(10):
    os_[:, k:].zero_()
print(f"host zeroing of the fill distances (19.2 MB): {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms "
      f"({torch.get_num_threads()} threads)")
for ch in (2, 4, 8):
    f = lambda: ffps.hierarchical_sample_host(pinned, budgets, cfg, out=(oi, os_), chunks=ch,
                                              precision="f64")
    print(f"host pipeline, {ch} chunks: {timed(f):.3f} ms")
