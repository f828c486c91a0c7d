#!/usr/bin/env python
"""Strong-scaling shapes of the C5 FlashFPS greedy stage (50,000 candidates,
12,500 iterations): the clouds one GPU holds when the global batch of 64 is
split over 1/2/4/8 GPUs (64/32/16/8), under K1g with 1/2/4 CTAs per cloud,
binary32 and binary64-on-float (FFPS_F32_F64).  One JSON line per case:
median greedy-call time (CUDA events, K0 included), rounds and cycles per
round from the kernel counters."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17720_b200 as ffps  # noqa: E402
from paper_2604_17720_b200 import _device  # noqa: E402


def run(x, n, it, precision, reps=3):
    B = x.shape[0]
    ts = []
    out = None
    for r in range(reps + 1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out, _ = ffps.fps_batch(x[:, :n], it, precision=precision)
        e.record()
        torch.cuda.synchronize()
        if r:
            ts.append(s.elapsed_time(e))
    with _device.grid_stats() as gs:
        ffps.fps_batch(x[:, :n], it, precision=precision)
        torch.cuda.synchronize()
    st = gs.records[0][3].double()
    return float(np.median(ts)), out.indices.cpu(), float(st[:, 0].mean()), float(st[:, 1].mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, nargs="*", default=[8, 16, 32, 64])
    ap.add_argument("--n", type=int, default=50_000)
    ap.add_argument("--iters", type=int, default=12_500)
    ap.add_argument("--scheds", nargs="*", default=["grid@1", "grid@2", "grid@4", "grid@2/km8"])
    ap.add_argument("--precisions", nargs="*", default=["f64", "f32"])
    ap.add_argument("--cloud", choices=["uniform", "lidar"], default="uniform")
    ap.add_argument("--cloud-n", type=int, default=0,
                    help="LiDAR frame size (the candidates are its first n points); 0: 4 n")
    a = ap.parse_args()
    if a.cloud == "lidar":
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        frames = bench.make_clouds("lidar", max(a.batches), a.cloud_n or 4 * a.n, 0)
        x = torch.from_numpy(np.ascontiguousarray(frames[:, :a.n])).cuda()
    else:
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.rand((max(a.batches), a.n, 3), generator=g, device="cuda",
                       dtype=torch.float64).float()
    for B in a.batches:
        xb = x[:B].contiguous()
        for prec in a.precisions:
            ref = None
            for sc in a.scheds:
                name, _, km = sc.partition("/km")
                keep = os.environ.get("FFPS_GRID_KM")
                if km:
                    os.environ["FFPS_GRID_KM"] = km
                _device.set_schedule(name)
                try:
                    ms, order, rounds, cyc = run(xb, a.n, a.iters, prec)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"B": B, "sched": sc, "prec": prec, "error": str(e)[:120]}))
                    continue
                same = True if ref is None else bool(torch.equal(order, ref))
                ref = order if ref is None else ref
                print(json.dumps({"B": B, "n": a.n, "iters": a.iters, "sched": sc, "prec": prec,
                                  "ms": round(ms, 3), "rounds": rounds,
                                  "cycles_per_round": round(cyc / max(rounds, 1), 1),
                                  "same": same}), flush=True)
                if km:
                    os.environ.pop("FFPS_GRID_KM", None)
                    if keep is not None:
                        os.environ["FFPS_GRID_KM"] = keep
            _device.set_schedule("auto")


if __name__ == "__main__":
    main()
