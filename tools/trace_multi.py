#!/usr/bin/env python
"""Phase trace of K1g (multi-winner rounds), CTA 0: per round and warp
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
    ap.add_argument("--sched", default="grid@2",
                    choices=["grid", "grid@1", "grid@2", "grid@4"])
    ap.add_argument("--cloud", choices=["uniform", "lidar"], default="uniform")
    ap.add_argument("--cloud-n", type=int, default=200000)
    ap.add_argument("--precision", choices=["f32", "f64"], default="f32",
                    help="f64: binary64 arithmetic on the float coordinates (FFPS_F32_F64)")
    a = ap.parse_args()
    if a.cloud == "lidar":  # the bench's LiDAR frames, candidate prefix of n points
        import bench
        x = torch.from_numpy(bench.make_clouds("lidar", a.batch, a.cloud_n, 0)[:, :a.n].copy()).cuda()
    else:
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.rand((a.batch, a.n, 3), generator=g, device="cuda", dtype=torch.float64).float()
    W = 16 if a.sched.startswith("grid") else 8
    tr = torch.zeros((a.nw, a.iters, W), dtype=torch.int64, device="cuda")
    os.environ["FFPS_TRACE_MULTI" if a.sched.startswith("multi") else "FFPS_TRACE_GRID"] = \
        f"{tr.data_ptr()},{a.iters}"
    prev = _device.set_schedule(a.sched)
    B = a.batch
    order = torch.empty((B, a.iters), dtype=torch.int64, device="cuda")
    sel = torch.empty((B, a.iters), dtype=torch.float64 if a.precision == "f64" else x.dtype,
                      device="cuda")
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
    names = (["bound", "reeval", "topk", "merge+barriers"] if a.sched.startswith("multi") else
             ["flag", "reeval", "candidates", "merge+barriers"])
    ph = np.stack([t[:, :, i + 1] - t[:, :, i] for i in range(4)], -1)
    for lo, hi in [(1, max(2, R // 10)), (R // 10, R)]:
        sl = slice(lo, hi)
        tot = t[0, sl, 4] - t[0, sl, 0]
        flagged = (t[0, sl, 6] & 0xffffffff) if a.sched.startswith("grid") else t[:, sl, 6].sum(0)
        if a.sched.startswith("grid"):
            info = t[0, sl, 7]
            print(f"   candidates per round (warp 0) {(t[0, sl, 6] >> 32).mean():.1f}, "
                  f"bucket groups {(info[0] >> 1) & 0x7fffff}, hit groups per warp-round "
                  f"{np.mean([(t[w, sl, 7] >> 24).mean() for w in range(t.shape[0])]):.1f}")
        print(f"rounds [{lo},{hi}): cycles/round median {np.median(tot):.0f}, winners/round "
              f"{nsel[sl].mean():.2f}, flagged/round {flagged.mean():.1f}" +
              (f", full-scan rounds {(t[0, sl, 7] & 1).mean():.2f}" if a.sched.startswith("grid") else ""))
        for i, nm in enumerate(names):
            v = ph[:, sl, i]
            print(f"   {nm:15s} mean {v.mean():7.0f}  max-warp mean {v.max(0).mean():7.0f}")
        if W == 16:  # warp 0 sub-steps of phase D (0 = not reached / not traced)
            d = t[0, sl, 8:16].astype(np.float64)
            t3 = t[0, sl, 3].astype(np.float64)
            marks = ["B3", "R", "B4", "select", "push", "wait", "merge", "chain"]
            prev = t3
            out = []
            for i, m in enumerate(marks):
                ok = d[:, i] > 0
                if ok.any():
                    out.append(f"{m} {np.median(d[ok, i] - prev[ok]):.0f}")
                    prev = np.where(ok, d[:, i], prev)
            out.append(f"tail {np.median(t[0, sl, 4] - prev):.0f}")
            print("   D (warp 0, median cycles from the previous mark): " + ", ".join(out))
    if a.sched.startswith("grid"):
        # where the loop's cycles go: round 0 (the seed's full scan), the early
        # rounds, the rest; general-path rounds (warp 0's ncand bit 16)
        tot = (t[0, :, 4] - t[0, :, 0]).astype(np.float64)
        gen = ((t[0, :, 6] >> 48) & 1).astype(bool)
        print(f"loop cycles (CTA 0, rank 0): total {tot.sum():.0f}, mean {tot.mean():.0f} per round")
        for lo, hi in [(0, 1), (1, 10), (10, R // 10), (R // 10, R)]:
            if hi <= lo:
                continue
            seg = tot[lo:hi]
            print(f"   rounds [{lo},{hi}): {seg.sum() / tot.sum():6.1%} of the cycles, mean "
                  f"{seg.mean():.0f}, winners {nsel[lo:hi].sum()}")
        if gen.any():
            nct = (t[0, :, 6] >> 32) & 0xffff
            ng_ = nct[gen]
            print(f"   general-path rounds: {gen.sum()} ({tot[gen].sum() / tot.sum():.1%} of the "
                  f"cycles, mean {tot[gen].mean():.0f}); keys >= tau2: <= 32 {(ng_ <= 32).sum()}, "
                  f"33-64 {((ng_ > 32) & (ng_ <= 64)).sum()}, > 64 (one winner) {(ng_ > 64).sum()}; "
                  f"winners/round {nsel[gen].mean():.2f} vs {nsel[~gen].mean():.2f}")


if __name__ == "__main__":
    main()
