#!/usr/bin/env python
"""Phase trace of K1m (multi-winner rounds), CTA 0: per round and warp
{start, bound test, re-evaluation, warp top-K, after merge}, winners taken
per round and flagged buckets of the warp."""
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
    ap.add_argument("--sched", default="multi", choices=["multi", "grid"])
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((a.batch, a.n, 3), generator=g, device="cuda", dtype=torch.float64).float()
    tr = torch.zeros((a.nw, a.iters, 8), dtype=torch.int64, device="cuda")
    os.environ["FFPS_TRACE_MULTI" if a.sched == "multi" else "FFPS_TRACE_GRID"] = \
        f"{tr.data_ptr()},{a.iters}"
    prev = _device.set_schedule(a.sched)
    B = a.batch
    order = torch.empty((B, a.iters), dtype=torch.int64, device="cuda")
    sel = torch.empty((B, a.iters), dtype=x.dtype, device="cuda")
    seeds = torch.zeros(B, dtype=torch.int64, device="cuda")
    _device.greedy(x, a.n, a.iters, seeds, order, sel)
    torch.cuda.synchronize()
    _device.set_schedule(prev)
    t = tr.cpu().numpy()
    R = int((t[0, :, 0] != 0).sum())
    t = t[:, :R, :]
    nsel = t[0, :, 5]
    print(f"rounds {R} for {a.iters} iterations: {nsel.sum() + 1} winners, "
          f"{(nsel.sum()) / R:.2f} per round")
    names = (["bound", "reeval", "topk", "merge+barriers"] if a.sched == "multi" else
             ["flag", "reeval", "candidates", "merge+barriers"])
    ph = np.stack([t[:, :, i + 1] - t[:, :, i] for i in range(4)], -1)
    for lo, hi in [(1, max(2, R // 10)), (R // 10, R)]:
        sl = slice(lo, hi)
        tot = t[0, sl, 4] - t[0, sl, 0]
        flagged = t[0, sl, 6] if a.sched == "grid" else t[:, sl, 6].sum(0)
        if a.sched == "grid":
            info = t[0, sl, 7]
            print(f"   oversize buckets {(info[0] >> 1) & 0x7fffff}, cell entries per point "
                  f"(warps with a point) {np.mean([((t[w, sl, 7] >> 24) / 2).mean() for w in range(t.shape[0])]):.1f}")
        print(f"rounds [{lo},{hi}): cycles/round median {np.median(tot):.0f}, winners/round "
              f"{nsel[sl].mean():.2f}, flagged/round {flagged.mean():.1f}" +
              (f", full-scan rounds {t[0, sl, 7].mean():.2f}" if a.sched == "grid" else ""))
        for i, nm in enumerate(names):
            v = ph[:, sl, i]
            print(f"   {nm:15s} mean {v.mean():7.0f}  max-warp mean {v.max(0).mean():7.0f}")


if __name__ == "__main__":
    main()
