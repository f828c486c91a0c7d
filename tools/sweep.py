#!/usr/bin/env python
"""Time K1 (the greedy kernel) for one (batch, n, iters) shape under every
kernel configuration forced through FFPS_FORCE_PLAN, plus the planner's own
choice.  CUDA events on the launching stream, 1 warm-up + median of 3.

    python tools/sweep.py --batch 64 --n 50000 --iters 12500 \\
        --plans 256,14,36,4 128,28,72,4 ...
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17720_b200 import _device, _native  # noqa: E402


def run(x, n, iters, reps):
    B = x.shape[0]
    order = torch.empty((B, iters), dtype=torch.int64, device=x.device)
    sel = torch.empty((B, iters), dtype=x.dtype, device=x.device)
    seeds = torch.zeros(B, dtype=torch.int64, device=x.device)
    _device.greedy(x, n, iters, seeds, order, sel)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        _device.greedy(x, n, iters, seeds, order, sel)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts)), order


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--cloud-n", type=int, default=None)
    ap.add_argument("--iters", type=int, default=12500)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--plans", nargs="*", default=[])
    a = ap.parse_args()
    dt = getattr(torch, a.dtype)
    N = a.cloud_n or a.n
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((a.batch, N, 3), generator=g, device="cuda", dtype=torch.float64).to(dt)
    units = a.batch * a.n * (a.iters - 1)
    import subprocess
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    ref = None
    for plan in [""] + a.plans:
        os.environ["FFPS_FORCE_PLAN"] = plan
        try:
            ms, order = run(x, a.n, a.iters, a.reps)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"plan": plan or "auto", "error": str(e)[:200]}), flush=True)
            continue
        if ref is None:
            ref = order
        same = bool(torch.equal(order, ref))
        info = _native.plan(_native.F32 if dt == torch.float32 else _native.F64, a.n, a.batch) \
            if not plan else {}
        print(json.dumps({"plan": plan or "auto", "ms": round(ms, 4), "idle_clk": clk,
                          "ns_per_iter": round(ms * 1e6 / a.iters, 1),
                          "gunits_per_s": round(units / ms / 1e6, 1), "same_as_auto": same,
                          **({"auto": info} if info else {})}), flush=True)
    os.environ.pop("FFPS_FORCE_PLAN", None)


if __name__ == "__main__":
    main()
