#!/usr/bin/env python
"""C5 FPS-Prune layer 1 (64 clouds x 200K, m1 = 50,000, p = 0.75) with the
slice fill (K2) and the seeded random fill (K2r): ms per batch, and the fill
kernels alone; CUDA events, median of 5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402
from paper_2604_17720_b200 import _device  # noqa: E402

B, N, m1 = 64, 200000, 50000
x = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).cuda()


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


for mode in (ffps.FillMode.DETERMINISTIC_SLICE, ffps.FillMode.SEEDED_RANDOM):
    cfg = ffps.PruneConfig(p=0.75, fill_mode=mode, rng_seed=3)
    ms = timed(lambda: ffps.fps_prune_batch(x, m1, cfg))
    out, _ = ffps.fps_prune_batch(x, m1, cfg)
    k = out.fill_boundary
    order, sel = out.indices.clone(), out.selection_dist2.clone()
    if mode is ffps.FillMode.DETERMINISTIC_SLICE:
        fill = lambda: _device.fill_slice(order, sel, k, m1)  # noqa: E731
    else:
        fill = lambda: _device.fill_random(order, sel, N, k, m1, 3)  # noqa: E731
    print(f"{mode.value}: layer 1 {ms:.2f} ms, fill kernel {timed(fill):.3f} ms "
          f"({m1 - k} fill entries per cloud)", flush=True)
