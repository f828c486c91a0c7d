#!/usr/bin/env python
"""Phase trace of K1 (streaming cluster kernel), cluster 0: per iteration and
warp of every rank the %clock64 stamps {start, update done, record pushed,
records arrived, end}.  Prints per-phase cycle statistics."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device, _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--iters", type=int, default=12500)
    a = ap.parse_args()
    plan = _native.plan(_native.F32, a.n, a.batch)
    C, NW = plan["cluster"], plan["threads"] // 32
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((a.batch, a.n, 3), generator=g, device="cuda", dtype=torch.float64).float()
    tr = torch.zeros((C * NW, a.iters, 8), dtype=torch.int64, device="cuda")
    os.environ["FFPS_TRACE_STREAM"] = f"{tr.data_ptr()},{a.iters}"
    prev = _device.set_schedule("stream")
    B = a.batch
    order = torch.empty((B, a.iters), dtype=torch.int64, device="cuda")
    sel = torch.empty((B, a.iters), dtype=x.dtype, device="cuda")
    seeds = torch.zeros(B, dtype=torch.int64, device="cuda")
    _device.greedy(x, a.n, a.iters, seeds, order, sel)
    torch.cuda.synchronize()
    _device.set_schedule(prev)
    t = tr.cpu().numpy()[:, 1:, :]
    names = ["update", "winner+push", "wait", "combine+mark"]
    ph = np.stack([t[:, :, i + 1] - t[:, :, i] for i in range(4)], -1)
    print(f"plan {plan}; warps traced {C * NW}")
    K = t.shape[1]
    for lo, hi in [(0, K // 10), (K // 10, K)]:
        sl = slice(lo, hi)
        tot = t[:, sl, 4] - t[:, sl, 0]
        print(f"iters [{lo},{hi}): cycles/iter median {np.median(tot):.0f}")
        for i, nm in enumerate(names):
            v = ph[:, sl, i]
            print(f"   {nm:13s} mean {v.mean():7.0f}  median {np.median(v):7.0f}  max-warp mean {v.max(0).mean():7.0f}")
    it = np.diff(t[0, :, 0])
    print("iteration period (rank 0 warp 0) median", np.median(it))


if __name__ == "__main__":
    main()
