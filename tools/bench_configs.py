#!/usr/bin/env python
"""Every BASELINE.json config on one GPU, both greedy schedules: ms/step,
clouds/s, ns per greedy iteration, FlashFPS vs exhaustive speedups.
CUDA events, 2 warm-up + median of 5 (heavy exhaustive arms: 1 + 3)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402
from paper_2604_17720_b200 import _device  # noqa: E402

CONFIGS = [
    # name, B, N, budgets, p values for FlashFPS
    ("C1 exhaustive fps", 1, 4096, (1024,), ()),
    ("C2 FPS-Prune 4-stage", 16, 24000, (6000, 1500, 375, 93), (0.25, 0.5, 0.75)),
    ("C3 PointNeXt-L S3DIS prune+cache", 8, 100000, (25000, 6250, 1562, 390), (0.75,)),
    ("C4 LiDAR-frame 4-stage", 32, 300000, (75000, 18750, 4687, 1171), (0.75,)),
    ("C5 scaling batch", 64, 200000, (50000, 12500, 3125, 781), (0.75,)),
]


def timeit(fn, warm, reps):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("clouds", nargs="*", default=["uniform"])
    ap.add_argument("--scheds", nargs="*", default=["auto", "stream"])
    ap.add_argument("--configs", nargs="*", default=None, help="name prefixes, e.g. C5")
    ap.add_argument("--precision", choices=["f64", "f32"], default="f64",
                    help="f64: the reference's binary64 on the fp32 clouds (FFPS_F32_F64)")
    a = ap.parse_args()
    for kind in a.clouds:
        for name, B, N, budgets, ps in CONFIGS:
            if kind == "lidar" and N < 100000:
                continue
            if a.configs and not any(name.startswith(c) for c in a.configs):
                continue
            x = torch.from_numpy(bench.make_clouds(kind, B, N, 0)).cuda()
            for sched in a.scheds:
                prev = _device.set_schedule(sched)
                try:
                    heavy = N >= 100000 and sched in ("stream", "bucket")
                    ex = timeit(lambda: ffps.hierarchical_sample_batch(
                        x, budgets, ffps.PruneConfig(p=0.0), 0, False, precision=a.precision),
                        1 if heavy else 2, 3 if heavy else 5)
                    rec = {"config": name, "cloud": kind, "B": B, "N": N, "schedule": sched,
                           "precision": a.precision,
                           "exhaustive_ms": ex, "exhaustive_clouds_per_s": B / ex * 1e3}
                    for p in ps:
                        fl = timeit(lambda: ffps.hierarchical_sample_batch(
                            x, budgets, ffps.PruneConfig(p=p), 0, True, precision=a.precision),
                            2, 5)
                        k = ffps.PruneConfig(p=p).kernel_budget(budgets[0])
                        rec[f"flash_p{p}_ms"] = fl
                        rec[f"flash_p{p}_clouds_per_s"] = B / fl * 1e3
                        rec[f"flash_p{p}_ns_per_iter"] = fl * 1e6 / k
                        rec[f"speedup_p{p}_vs_exhaustive"] = ex / fl
                    print(json.dumps(rec), flush=True)
                finally:
                    _device.set_schedule(prev)


if __name__ == "__main__":
    main()
