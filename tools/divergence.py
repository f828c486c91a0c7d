#!/usr/bin/env python
"""Every divergence of binary32 from the reference's binary64, per cloud, at
the BASELINE configurations (north star: "every divergence is reported").

For C2-C5 (uniform and LiDAR-like clouds) runs the FlashFPS layer 1 (greedy
prefix of k points) and the exhaustive layer 1 in binary32 and in binary64
(FFPS_F32_F64: bit-identical to the reference on the fp32 clouds) and writes
per-cloud first divergent position, mismatched positions and the overlap of
the selected sets (bench.divergence).  One JSON line per (config, cloud kind,
pipeline)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_17720_b200 as ffps  # noqa: E402

CONFIGS = [("C2", 16, 24_000), ("C3", 8, 100_000), ("C4", 32, 300_000), ("C5", 64, 200_000)]


def main():
    kinds = sys.argv[1:] or ["uniform", "lidar"]
    for kind in kinds:
        for name, B, N in CONFIGS:
            budgets = bench.BUDGETS[N]
            x = torch.from_numpy(bench.make_clouds(kind, B, N, 0)).cuda()
            c, k = bench.stage_units(N, budgets, 0.75, True)[0]
            for pipe, cfg, cache, n_sel, cand in (("flash_layer1_greedy", 0.75, True, k, c),
                                                  ("exhaustive_layer1", 0.0, False, budgets[0], N)):
                a, _, _ = ffps.hierarchical_sample_batch(x, budgets, ffps.PruneConfig(p=cfg), 0,
                                                         cache, precision="f64")
                b, _, _ = ffps.hierarchical_sample_batch(x, budgets, ffps.PruneConfig(p=cfg), 0,
                                                         cache, precision="f32")
                d = bench.divergence(a[0].indices[:, :n_sel], b[0].indices[:, :n_sel], cand)
                firsts = [f for f in d["first_divergence"] if f >= 0]
                print(json.dumps({"config": name, "cloud": kind, "pipeline": pipe, "B": B, "N": N,
                                  "k": n_sel, "identical_clouds": d["identical_clouds"],
                                  "earliest_divergence": min(firsts) if firsts else None,
                                  "mean_mismatched": sum(d["mismatched_positions"]) / B,
                                  "min_set_overlap": min(d["set_overlap"]), **d}), flush=True)


if __name__ == "__main__":
    main()
