#!/usr/bin/env python
"""Phase trace of K1b (bucketed kernel), CTA 0: per iteration and warp the
%clock64 stamps {start, bound test done, re-evaluation done, argmax done,
barrier passed, end} and the number of flagged buckets the warp owned.
Prints per-phase cycle statistics over iteration ranges."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--iters", type=int, default=12500)
    ap.add_argument("--nw", type=int, default=16)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((a.batch, a.n, 3), generator=g, device="cuda", dtype=torch.float64).float()
    tr = torch.zeros((a.nw, a.iters, 8), dtype=torch.int64, device="cuda")
    os.environ["FFPS_TRACE_BUCKET"] = f"{tr.data_ptr()},{a.iters}"
    os.environ["FFPS_ALGO"] = "bucket"
    B = a.batch
    order = torch.empty((B, a.iters), dtype=torch.int64, device="cuda")
    sel = torch.empty((B, a.iters), dtype=x.dtype, device="cuda")
    seeds = torch.zeros(B, dtype=torch.int64, device="cuda")
    _device.greedy(x, a.n, a.iters, seeds, order, sel)
    torch.cuda.synchronize()
    t = tr.cpu().numpy()[:, 1:, :]  # (warps, iters-1, 8)
    names = ["bound", "reeval", "argmax", "barrier", "final"]
    ph = np.stack([t[:, :, i + 1] - t[:, :, i] for i in range(5)], -1)  # (w, k, 5)
    tot = t[:, :, 5] - t[:, :, 0]
    nf = t[:, :, 6]
    K = t.shape[1]
    for lo, hi in [(0, 100), (100, 1000), (1000, K // 2), (K // 2, K)]:
        sl = slice(lo, hi)
        print(f"iters [{lo},{hi}): total cycles/iter median {np.median(tot[0, sl]):.0f}; "
              f"flagged/iter (all warps) mean {nf[:, sl].sum(0).mean():.1f}, "
              f"max per warp mean {nf[:, sl].max(0).mean():.2f}")
        for i, nm in enumerate(names):
            v = ph[:, sl, i]
            print(f"   {nm:8s} mean over warps {v.mean():7.0f}  max-warp mean {v.max(0).mean():7.0f}")
    it = np.diff(t[0, :, 0])
    print("iteration period (warp 0) median", np.median(it), "mean", it.mean())


if __name__ == "__main__":
    main()
