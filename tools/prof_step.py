import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_2604_17720_b200 as ffps
B, N, budgets = 64, 200000, (50000, 12500, 3125, 781)
x = torch.from_numpy(bench.make_clouds("uniform", B, N, 0)).cuda()
cfg = ffps.PruneConfig(p=0.75)
for _ in range(3):
    ffps.hierarchical_sample_batch(x, budgets, cfg, 0, True, precision="f64")
torch.cuda.synchronize()
# time to first kernel: a marker kernel before, events
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        torch.cuda.synchronize()
        ffps.hierarchical_sample_batch(x, budgets, cfg, 0, True, precision="f64")
        torch.cuda.synchronize()
ev = [e for e in prof.events()]
# print kernel events with their start offsets
ks = sorted([e for e in ev if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
cs = sorted([e for e in ev if e.device_type.name == "CPU"], key=lambda e: e.time_range.start)
t0 = cs[0].time_range.start
for e in ks[:40]:
    print(f"GPU {e.name[:60]:60s} start {(e.time_range.start - t0)/1e3:9.3f} ms dur {(e.time_range.end - e.time_range.start)/1e3:8.3f}")
for e in cs[:60]:
    if (e.time_range.end - e.time_range.start) > 5:
        print(f"CPU {e.name[:60]:60s} start {(e.time_range.start - t0)/1e3:9.3f} ms dur {(e.time_range.end - e.time_range.start)/1e3:8.3f}")
