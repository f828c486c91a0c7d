#!/usr/bin/env python
"""End-to-end C5 FlashFPS (pinned host clouds -> host indices) for several
chunk counts of hierarchical_sample_host: ms per batch, median of 5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402

B, N, budgets = 64, 200000, (50000, 12500, 3125, 781)
pinned = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).pin_memory()
cfg = ffps.PruneConfig(p=0.75)
oi = torch.empty((B, budgets[0]), dtype=torch.int64).pin_memory()
prec = os.environ.get("FFPS_E2E_PRECISION", "f64")
os_ = torch.empty((B, budgets[0]),
                  dtype=torch.float64 if prec == "f64" else torch.float32).pin_memory()
for ch in [int(c) for c in (sys.argv[1:] or ["1", "2", "4", "8", "16"])]:
    for _ in range(3):
        ffps.hierarchical_sample_host(pinned, budgets, cfg, out=(oi, os_), chunks=ch,
                                      precision=prec)
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        ffps.hierarchical_sample_host(pinned, budgets, cfg, out=(oi, os_), chunks=ch,
                                      precision=prec)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"chunks {ch}: {np.median(ts):.3f} ms  ({B / np.median(ts) * 1e3:.0f} clouds/s)", flush=True)
