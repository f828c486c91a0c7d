#!/usr/bin/env python
"""C5 FlashFPS 4-stage (64 clouds x 200K, p = 0.75 + cache) in binary32 and in
binary64 (the reference's precision, bit-exact vs the unmodified reference):
ms per batch and clouds/s, CUDA events, median of 5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402

B, N, budgets = 64, 200000, (50000, 12500, 3125, 781)
x32 = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).cuda()
for name, x in (("f32", x32), ("f64", x32.double())):
    for cfg, cache, label in ((ffps.PruneConfig(p=0.75), True, "flash"),
                              (ffps.PruneConfig(p=0.0), False, "exhaustive")):
        run = lambda: ffps.hierarchical_sample_batch(x, budgets, cfg, 0, cache)  # noqa: E731
        for _ in range(2):
            run()
        ts = []
        for _ in range(5 if label == "flash" else 3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            run()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = float(np.median(ts))
        print(f"{name} {label}: {ms:.2f} ms per 64 clouds, {B / ms * 1e3:.0f} clouds/s", flush=True)
