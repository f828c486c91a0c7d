#!/usr/bin/env python
"""One small invocation of every kernel family, for compute-sanitizer
(tools/gpu_sanitize.sh): K1 (stream, cluster/DSMEM/mbarrier), K1s, K0 + K1b,
K0 + K1g with 1/2/4 CTAs per cloud (st.async + mbarrier exchange)
in binary32, binary64 and binary64-on-float, K2/K2r fills and K5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17720_b200 as ffps  # noqa: E402
from paper_2604_17720_b200 import _device  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)
x32 = torch.from_numpy(rng.random((2, 3000, 3)).astype(np.float32)).cuda()
x64 = x32.double()
runs = []
for sched in ("stream", "small", "bucket", "grid@1", "grid@2", "grid@4"):
    for name, x, prec in (("f32", x32, None), ("f64", x64, None), ("f32_f64", x32, "f64")):
        runs.append((f"{sched}/{name}", sched, x, prec))
for tag, sched, x, prec in runs:
    if which != "all" and not tag.startswith(which):
        continue
    prev = _device.set_schedule(sched)
    try:
        s, _ = ffps.fps_batch(x, 300, precision=prec)
        torch.cuda.synchronize()
    finally:
        _device.set_schedule(prev)
    print(tag, "ok", int(s.indices[0, 299]))
if which in ("all", "fill"):
    ffps.hierarchical_sample_batch(x32, (1200, 300, 75), ffps.PruneConfig(p=0.5))
    ffps.fps_prune_batch(x32, 1200, ffps.PruneConfig(p=0.5, fill_mode=ffps.FillMode.SEEDED_RANDOM,
                                                     rng_seed=3))
    ffps.coverage_d2_batch(x32, s.indices)
    torch.cuda.synchronize()
    print("fill/coverage ok")
